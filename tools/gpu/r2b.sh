cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m "gpu and slow" -x -q -p no:cacheprovider --durations=0 > gpurun_out/r2b_slow.log 2>&1; echo "slow rc=$?"
tail -25 gpurun_out/r2b_slow.log
for w in c2 ens-c2-b128 ftr-c2-b128 c4-64 c4-256 c5; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r2b_$w.json 2> gpurun_out/r2b_$w.err; echo "$w rc=$?"
  tail -c 900 gpurun_out/r2b_$w.json; echo
done
