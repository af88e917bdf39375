#!/bin/bash
# A/B of two builds of the library on one box (SS_LIB_PATH), alternating runs
# of the headline bench: tools/ab_bench.sh libA.so libB.so rounds [extra bench args]
A=$1; B=$2; N=${3:-2}; shift 3; EXTRA="$@"
mkdir -p gpurun_out/ab
for r in $(seq 1 $N); do
  for L in $A $B; do
    SS_LIB_PATH=$L timeout 300 python bench.py --no-configs --no-cpu-baseline --steps 30 $EXTRA > gpurun_out/ab/out.json 2>/dev/null
    python -c "import json,sys;d=json.loads(open('gpurun_out/ab/out.json').read().strip().splitlines()[-1]);print(sys.argv[1], d['value'], d['e2e']['value'], d['config']['stage_ms_median'])" $L
  done
done
