#!/bin/bash
# A/B of library variants on one box: tools/gpu_ab.sh TAG VARIANT...   (VARIANT "base" = libdiffreg.so,
# "pair" = libdiffreg.so with DR_WINDOW=0, other names = libdiffreg_<name>.so via DR_LIB_VARIANT)
set -u
TAG=$1; shift
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
for V in "$@"; do
  if [ "$V" = "base" ]; then E=""; elif [ "$V" = "pair" ]; then E="DR_WINDOW=0"; else E="DR_LIB_VARIANT=$V"; fi
  env $E timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --profile-out gpurun_out/${TAG}_prof_$V.json > gpurun_out/${TAG}_bench_$V.json 2> gpurun_out/${TAG}_bench_$V.err
  echo "== $V rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${TAG}_bench_$V.json'));print(round(d['value'],1),'mv/s', round(d['matvec_only_ms'],3),'ms/mv')" 2>/dev/null)"
  python tools/show_prof.py gpurun_out/${TAG}_prof_$V.json 2>/dev/null | grep -E "step|sl_" | head -12
done
