#!/bin/bash
# per-layer conv timings: current build vs lib/alt (SS_LIB_PATH)
ALT=$PWD/paper_2301_00750_b200/lib/alt/libstreamstab_b200.so
for cfg in "SS_NONE=1" "SS_LIB_PATH=$ALT" "SS_NONE=1" "SS_LIB_PATH=$ALT"; do
  out=$(env $cfg SS_FLOW_PROFILE=1 timeout 120 python tools/flow_prof.py fp32 2>&1 | sed -n '/measured call/,$p' | grep -E "pyr1b|est3_1 |est3_2|est4_1 |total" | awk '{print $3"="$4}' | tr '\n' ' ')
  echo "[${cfg:0:12}] $out"
done
