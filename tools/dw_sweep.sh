for px in 4 2 1 8; do
  touch paper_2301_00750_b200/csrc/flownet_kernels.cu
  make -s -C paper_2301_00750_b200/csrc EXTRA="-DDW_PX_OVERRIDE=$px" > /dev/null 2>&1
  echo "DW_PX=$px: $(SS_FLOW_PROFILE=1 python tools/flow_prof.py fp32 2>&1 | grep -E '_dw' | tail -6 | awk '{print $4}' | tr '\n' ' ') | $(timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"])')"
done
