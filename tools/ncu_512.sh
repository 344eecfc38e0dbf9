#!/bin/bash
# ncu --set full of the 512^3 column passes (isochoric kind-8 middle, ColDivPass, non-isochoric kind-0 middle)
set -u
TAG=$1
mkdir -p gpurun_out
for spec in "MiddlePass<double, float, .int.512, .int.8:0" "ColDivPass<float, .int.512:0" "MiddlePass<double, float, .int.512, .int.0:0"; do
  K=${spec%:*}; S=${spec##*:}; N=$(echo "$K" | tr -c 'A-Za-z0-9' '_')
  timeout 900 ncu --set full --metrics lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:${K}" -s $S -c 1 -o gpurun_out/prof_${TAG}_$N python tools/prof_config4b.py > gpurun_out/ncu_${TAG}_$N.log 2>&1
  R=gpurun_out/prof_${TAG}_$N.ncu-rep
  if [ -f $R ]; then
    python tools/ncu_summary.py $R > gpurun_out/summary_${TAG}_$N.txt 2>&1; head -24 gpurun_out/summary_${TAG}_$N.txt
    ncu -i $R --page raw --csv > gpurun_out/raw_${TAG}_$N.csv 2>/dev/null
    ncu -i $R --page details > gpurun_out/details_${TAG}_$N.txt 2>/dev/null
    rm -f $R
  else grep -i "warn\|error" gpurun_out/ncu_${TAG}_$N.log | head -3; fi
done
