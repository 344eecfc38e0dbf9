#!/bin/bash
# A/B of the spectral-overlap experiment (DR_OVERLAP 1/2, DR_GATHER_PAD) on one box: tools/ab_overlap.sh TAG
# (the DR_OVERLAP=2 and DR_GATHER_PAD knobs were experiment builds, removed after the measurement in
# profiles/ab_overlap_r2s.txt; DR_OVERLAP=1 remains)
set -u
TAG=$1
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for E in "DR_GRAPHS=0" "DR_GRAPHS=0 DR_OVERLAP=1" "DR_GRAPHS=0 DR_OVERLAP=2" "DR_GRAPHS=0 DR_OVERLAP=2 DR_GATHER_PAD=26000" "DR_GRAPHS=0 DR_OVERLAP=1 DR_GATHER_PAD=26000" "DR_OVERLAP=2" "" ; do
  N=$(echo "x$E" | tr -c 'A-Za-z0-9' '_')
  env $E timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_$N.json 2> gpurun_out/${TAG}_$N.err
  echo "== [$E] rc=$? $(python -c "import json;d=json.load(open('gpurun_out/${TAG}_$N.json'));print(round(d['value'],1),'mv/s', round(d['matvec_only_ms'],3),'ms/mv', d['clocks']['sm_mhz'])" 2>/dev/null)"
done
