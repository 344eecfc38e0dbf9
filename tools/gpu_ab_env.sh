#!/bin/bash
# A/B of environment settings on one box: tools/gpu_ab_env.sh TAG "ENV=..." "ENV=..." ...  ("-" = defaults)
set -u
TAG=$1; shift
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
i=0
for E in "$@"; do
  [ "$E" = "-" ] && E=""
  env $E timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --profile-out gpurun_out/${TAG}_prof_$i.json > gpurun_out/${TAG}_bench_$i.json 2> gpurun_out/${TAG}_bench_$i.err
  echo "== [$E] rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench_$i.json'));print(round(d['value'],1),'mv/s', round(d['matvec_only_ms'],3),'ms/mv')" 2>/dev/null)"
  python tools/show_prof.py gpurun_out/${TAG}_prof_$i.json 2>/dev/null | grep -E "step|row_|col_" | head -14
  i=$((i+1))
done
