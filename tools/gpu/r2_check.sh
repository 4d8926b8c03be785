#!/usr/bin/env bash
# Round-2 checkpoint: full GPU test suite, smoke, default bench + a few workloads.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2c
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2c/smi.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider --durations=15 > gpurun_out/r2c/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2c/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c/smoke.log 2>&1; echo "smoke rc=$?"
for w in c1 c2 c3 c4-64 c4-256 c5 ens-c2 ens-c2-b128 ftr-c2-b128 oop-c2; do
  timeout 300 python bench.py --workload "$w" > "gpurun_out/r2c/bench_$w.json" 2> "gpurun_out/r2c/bench_$w.err"
  echo "$w rc=$?"; cut -c1-400 gpurun_out/r2c/bench_$w.json
done
timeout 600 python bench.py --impl reference > gpurun_out/r2c/bench_ref.json 2> gpurun_out/r2c/bench_ref.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/r2c/bench_ref.json
