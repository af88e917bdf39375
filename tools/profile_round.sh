#!/bin/bash
# GPU-side profiling recipe for profiles/ (run under gpurun from the repo root):
#   launch list of the default bench (fp32 flow), then one `ncu --set full`
#   capture per hot kernel: conv est3_1 (fp32 and bf16), corr L3, solver pass,
#   K1 presolve.  Summaries: python profiles/summarize.py {launches|full} <file>
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py --steps 2 --warmup 3 > $OUT/bench_plain.json 2> $OUT/bench_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_fp32.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
# stateless flow: k_conv_tc3 launch 60 = est3_1 of the first flow (after two 21-launch pyramids + est6..est4)
ncu --set full --import-source on --clock-control none --kernel-name regex:k_conv_tc3 --launch-skip 60 --launch-count 1 \
    -o $OUT/conv_est3_1_fp32 python tools/flow_prof.py fp32 > $OUT/ncu_c1.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:k_conv_tc3 --launch-skip 60 --launch-count 1 \
    -o $OUT/conv_est3_1_bf16 python tools/flow_prof.py bf16 > $OUT/ncu_c2.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:k_corr --launch-skip 3 --launch-count 1 \
    -o $OUT/corr_l3 python tools/flow_prof.py fp32 > $OUT/ncu_c3.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:k_sgd_tma --launch-skip 40 --launch-count 1 \
    -o $OUT/solver_pass python bench.py --flow constant --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_s.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name regex:k_presolve --launch-skip 3 --launch-count 1 \
    -o $OUT/presolve python bench.py --flow constant --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_p.log 2>&1
ls -la $OUT
