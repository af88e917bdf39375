#!/bin/bash
# per-layer times of the flow network (SS_FLOW_PROFILE)
for p in fp32 fp32; do
  out=$(SS_FLOW_PROFILE=1 timeout 120 python tools/flow_prof.py $p 2>&1 | sed -n '/measured call/,$p' | grep -E "warp|prep|final|total" | awk '{print $3"="$4}' | tr '\n' ' ')
  echo "[$p] $out"
done
