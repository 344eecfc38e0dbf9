#!/bin/bash
# One GPU session: the -m gpu suite, then the default bench line.  Usage: tools/gpu_round.sh TAG [pytest -k expr]
set -u
TAG=$1; K=${2:-}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests/ -q -m gpu -k "$K" --tb=short > gpurun_out/${TAG}_pytest.log 2>&1
else
  timeout 1500 python -m pytest tests/ -q -m gpu --tb=short > gpurun_out/${TAG}_pytest.log 2>&1
fi
echo "pytest rc=$?"; tail -15 gpurun_out/${TAG}_pytest.log
if [ "${SKIPBENCH:-0}" != "1" ]; then
  timeout 900 python bench.py --profile-out gpurun_out/${TAG}_prof.json > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
  echo "bench rc=$?"; cut -c1-1500 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
fi
