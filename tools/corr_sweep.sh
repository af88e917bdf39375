set -e
for cs in "1 1" "2 2" "4 2" "4 4" "2 1"; do
  set -- $cs
  touch paper_2301_00750_b200/csrc/flownet_kernels.cu
  make -s -C paper_2301_00750_b200/csrc EXTRA="-DCR_CS_COARSE=$1 -DCR_CS_FINE=$2" > /dev/null 2>&1
  SS_FLOW_PROFILE=1 python tools/flow_prof.py fp32 > gpurun_out/prof_cs_$1_$2.txt 2>&1
  echo "CS $1 $2: $(sed -n '/measured call/,$p' gpurun_out/prof_cs_$1_$2.txt | grep -E 'corr|flow total' | awk '{print $3"="$4}' | tr '\n' ' ')"
done
