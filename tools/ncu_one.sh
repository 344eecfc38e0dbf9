#!/bin/bash
# ncu --set full of chosen kernels of one bench step: tools/ncu_one.sh TAG "regex:skip" ...  (env passes through)
set -u
TAG=$1; shift
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_${TAG}.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_${TAG}.log; exit 1; }
for spec in "$@"; do
  K=${spec%:*}; S=${spec##*:}; N=$(echo "$K" | tr -c 'A-Za-z0-9' '_')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:${K}" -s $S -c 1 -o gpurun_out/prof_${TAG}_$N $CMD > gpurun_out/ncu_full_${TAG}_$N.log 2>&1
  echo "ncu $K rc=$?"
  R=gpurun_out/prof_${TAG}_$N.ncu-rep
  [ -f $R ] && python tools/ncu_summary.py $R > gpurun_out/summary_${TAG}_$N.txt 2>&1 && head -30 gpurun_out/summary_${TAG}_$N.txt
done
