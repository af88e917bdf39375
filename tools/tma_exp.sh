#!/bin/bash
# timing experiments for the TMA conv (SS_TMA_DBG / SS_TMA_STAGES); results are
# numerically wrong for dbg != 0 -- timing only
for cfg in "0 0"; do
  set -- $cfg
  out=$(SS_TMA_DBG=$1 SS_TMA_STAGES=$2 SS_FLOW_PROFILE=1 timeout 120 python tools/flow_prof.py fp32 2>&1 | sed -n '/measured call/,$p' | grep -E "pyr1b|pyr2b|est3_1 |est3_2|est4_1 " | awk '{print $3"="$4}' | sort -u | tr '\n' ' ')
  echo "dbg=$1 stages=$2: $out"
done
