mkdir -p gpurun_out/ab4k
for r in 1; do for L in old new; do for sz in "1080 1920" "2160 3840" "720 1280"; do
SS_LIB_PATH=abtest/$L.so timeout 300 python tools/solver_bench.py $sz 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', d['size'], round(d['solve_ms_median'],4))"
done; done; done > gpurun_out/ab4k/ab.log 2>&1
