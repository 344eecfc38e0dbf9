#!/bin/bash
# ncu of the fused plane kernels: launch geometry + full sections
set -u
TAG=$1
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
for K in "k_plane_fwd<float, double>:2" "k_plane_inv<float>:2"; do
  N=$(echo "${K%:*}" | tr -c 'A-Za-z0-9' '_')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:${K%:*}" -s ${K##*:} -c 1 -o gpurun_out/prof_${TAG}_$N $CMD > gpurun_out/ncu_${TAG}_$N.log 2>&1
  R=gpurun_out/prof_${TAG}_$N.ncu-rep
  if [ -f $R ]; then
    python tools/ncu_summary.py $R > gpurun_out/summary_${TAG}_$N.txt 2>&1; head -24 gpurun_out/summary_${TAG}_$N.txt
    ncu -i $R --page details --csv 2>/dev/null | grep -E "Grid Size|Cluster|Block Size|Waves|DRAM Frequency|SM Frequency" | cut -c1-200
    ncu -i $R --page raw --csv > gpurun_out/raw_${TAG}_$N.csv 2>/dev/null
    rm -f $R
  else tail -3 gpurun_out/ncu_${TAG}_$N.log; fi
done
