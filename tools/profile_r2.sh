#!/bin/bash
# Round-2 GPU profiling recipe for profiles/ (run under gpurun from the repo
# root).  Every ncu command's plain run comes first in the same call (&&).
#   launch list of the default bench step (fp32 flow, headline config only);
#   ncu --set full: one k_sgd_v2 solver pass, K1 presolve, est3_1 (fp32 and
#   bf16, tools/conv_probe.py launches nothing else first), corr L3
#   (k_corr8); flow time against resolution; the full default bench.
set -x
OUT=gpurun_out/prof2
mkdir -p $OUT
B="python bench.py --steps 2 --warmup 3 --no-configs --no-e2e --no-cpu-baseline"
$B > $OUT/bench_plain.json 2> $OUT/bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_fp32.csv \
    $B > $OUT/ncu_launch.log 2>&1
S="python tools/solver_bench.py 1080 1920 6"
$S > $OUT/solver_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name regex:k_sgd_v2 --launch-skip 40 --launch-count 1 \
    -o $OUT/solver_pass $S > $OUT/ncu_s.log 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name regex:k_presolve --launch-skip 3 --launch-count 1 \
    -o $OUT/presolve $S > $OUT/ncu_p.log 2>&1
for p in fp32 bf16; do
  python tools/conv_probe.py $p > $OUT/conv_$p.log 2>&1 && \
  ncu --set full --import-source on --clock-control none --kernel-name regex:k_conv_tc3 --launch-skip 2 --launch-count 1 \
      -o $OUT/conv_est3_1_$p python tools/conv_probe.py $p > $OUT/ncu_c_$p.log 2>&1
done
F="python tools/flow_prof.py fp32"
$F > $OUT/flow_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name regex:k_corr8 --launch-skip 1 --launch-count 1 \
    -o $OUT/corr_l3 $F > $OUT/ncu_corr.log 2>&1
# flow time against resolution (the resolution-independent latency chain)
python tools/flow_scale.py fp32 > $OUT/flow_scale_fp32.txt 2>&1
python tools/flow_scale.py bf16 > $OUT/flow_scale_bf16.txt 2>&1
# the headline bench with every config
python bench.py > $OUT/bench_full.json 2> $OUT/bench_full.err
ls -la $OUT
