#!/bin/bash
# A/B of library builds (SS_LIB_PATH) on the solver alone at several sizes,
# same box: tools/ab_solver.sh libA.so libB.so [rounds]
A=$1; B=$2; N=${3:-1}
mkdir -p gpurun_out/ab_solver
for r in $(seq 1 $N); do for L in $A $B; do for sz in "1080 1920" "2160 3840" "720 1280"; do
  SS_LIB_PATH=$L timeout 300 python tools/solver_bench.py $sz 10 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], d['size'], round(d['solve_ms_median'], 4))" $L
done; done; done
