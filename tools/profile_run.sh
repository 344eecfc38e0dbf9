#!/bin/bash
# One GPU session: parity tests, the default bench line, then ncu (launch list + full captures).
# Env: KREGEX (kernel regex, default the inc-state gather), KSKIP (launches to skip), KCOUNT, SKIPTEST=1.
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
if [ "${SKIPTEST:-0}" != "1" ]; then
  python -m pytest tests/test_gpu_parity.py -q -m gpu --tb=short > gpurun_out/pytest_gpu_${TAG}.log 2>&1
  tail -3 gpurun_out/pytest_gpu_${TAG}.log
fi
python bench.py --profile-out gpurun_out/prof_${TAG}.json > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"; cut -c1-400 gpurun_out/bench_${TAG}.json
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${KREGEX:-EpiIncState}" -s ${KSKIP:-4} -c ${KCOUNT:-1} -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu rc=$?"
