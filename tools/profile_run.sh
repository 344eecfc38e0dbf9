#!/bin/bash
# One GPU session: parity tests, the default bench line, then ncu (launch list + full captures).
# Usage: tools/profile_run.sh TAG [kernel-regex ...]   (default regexes: the two matvec gathers)
# Env: KSKIP (matching launches to skip before capture, default 4), SKIPTEST=1, SKIPBENCH=1.
set -u
TAG=${1:-r1}
shift || true
KRES=("$@")
[ ${#KRES[@]} -eq 0 ] && KRES=("EpiIncState" "EpiAdjoint")
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi_${TAG}.txt 2>&1
lscpu > gpurun_out/lscpu_${TAG}.txt 2>&1
if [ "${SKIPTEST:-0}" != "1" ]; then
  timeout 1200 python -m pytest tests/ -q -m gpu --tb=short > gpurun_out/pytest_gpu_${TAG}.log 2>&1
  tail -3 gpurun_out/pytest_gpu_${TAG}.log
fi
if [ "${SKIPBENCH:-0}" != "1" ]; then
  timeout 900 python bench.py --profile-out gpurun_out/prof_${TAG}.json > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
  echo "bench rc=$?"; cut -c1-600 gpurun_out/bench_${TAG}.json
fi
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain_${TAG}.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_${TAG}.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:dr:: -c 800 --csv \
  --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "ncu launch rc=$?"
i=0
for K in "${KRES[@]}"; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:${K}" -s ${KSKIP:-4} -c 1 -o gpurun_out/prof_${TAG}_$i $CMD > gpurun_out/ncu_full_${TAG}_$i.log 2>&1
  echo "ncu full $K rc=$?"
  R=gpurun_out/prof_${TAG}_$i.ncu-rep
  if [ -f $R ]; then
    ncu -i $R --page details --csv > gpurun_out/details_${TAG}_$i.csv 2>/dev/null
    ncu -i $R --page raw --csv > gpurun_out/raw_${TAG}_$i.csv 2>/dev/null
    python tools/ncu_summary.py $R > gpurun_out/summary_${TAG}_$i.txt 2>&1
    [ "${KEEPREP:-0}" = "1" ] || rm -f $R
  fi
  i=$((i+1))
done
