#!/bin/bash
# Round-end evidence: GPU suite, default bench line, ncu launch list, --set full captures of the
# kernels the DESIGN/BASELINE tables cite.  Usage: tools/final_profile.sh TAG
set -u
TAG=${1:-final}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu --tb=short > gpurun_out/pytest_gpu_${TAG}.log 2>&1
tail -1 gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py --profile-out gpurun_out/prof_${TAG}.json > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_${TAG}.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -c 3000 --csv \
  -k regex:dr:: --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "ncu launch rc=$?"
# name regex : launches of that kernel to skip (setup / first matvec launches)
for spec in "EpiIncState:4" "EpiAdjoint:5" "MiddlePass<double:4" "RowR2cStaged:4" "RowC2rStaged:4" "ColFftPass<double:4"; do
  K=${spec%:*}; S=${spec##*:}; N=$(echo "$K" | tr -c 'A-Za-z0-9' '_')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:${K}" -s $S -c 1 -o gpurun_out/prof_${TAG}_$N $CMD > gpurun_out/ncu_full_${TAG}_$N.log 2>&1
  R=gpurun_out/prof_${TAG}_$N.ncu-rep
  if [ -f $R ]; then
    ncu -i $R --page raw --csv > gpurun_out/raw_${TAG}_$N.csv 2>/dev/null
    python tools/ncu_summary.py $R > gpurun_out/summary_${TAG}_$N.txt 2>&1
    rm -f $R
  fi
  echo "ncu full $K rc=$?"
done
