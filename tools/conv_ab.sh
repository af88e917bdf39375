#!/bin/bash
# per-layer conv timings: transposed thin-layer mode on / off (SS_CONV_TR)
for cfg in "SS_NONE=1" "SS_CONV_TR=0"; do
  out=$(env $cfg SS_FLOW_PROFILE=1 timeout 120 python tools/flow_prof.py fp32 2>&1 | sed -n '/measured call/,$p' | grep -E "pyr1b|pyr2b|pyr3b|est3_4|est3_5|est3_6|est4_4|ref5_pw|ref6_pw|ref7|total" | awk '{print $3"="$4}' | tr '\n' ' ')
  echo "[$cfg] $out"
done
