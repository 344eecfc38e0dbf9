set -u
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/w1_smi.txt 2>&1
timeout 900 python -m pytest tests/ -q -m gpu -x --tb=short > gpurun_out/w1_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/w1_pytest.log
for W in 0 1; do
  DR_WINDOW=$W timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --profile-out gpurun_out/w1_prof_$W.json > gpurun_out/w1_bench_$W.json 2> gpurun_out/w1_bench_$W.err; echo "bench W=$W rc=$?"
done
python tools/cmp_prof.py gpurun_out/w1_prof_0.json gpurun_out/w1_prof_1.json | head -30
