# round 2, GPU call 2: A/B of the PDL-safe GEMV / ENS scan against the round-1
# build on the same box; new ENS tensor-core batch + fused FTR split; slow tests timed
set -x
cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_ens.py tests/test_gpu_ftr.py tests/test_gpu_dist.py -x -q -p no:cacheprovider > gpurun_out/r2_tests.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/r2_tests.log
for i in 1 2; do
QPIR_LIB=$PWD/paper_2510_03631_b200/libqpir_r1.so python tools/sweep.py c2 -- --steps 2000 --warmup 20
python tools/sweep.py c2 -- --steps 2000 --warmup 20
done > gpurun_out/r2_ab.log 2>&1
QPIR_LIB=$PWD/paper_2510_03631_b200/libqpir_r1.so python tools/sweep.py ens-c2 >> gpurun_out/r2_ab.log 2>&1
python tools/sweep.py ens-c2 >> gpurun_out/r2_ab.log 2>&1
cat gpurun_out/r2_ab.log
python bench.py --workload ens-c2-b128 --no-cpu-baseline > gpurun_out/r2_ensb.json 2> gpurun_out/r2_ensb.err; tail -c 1500 gpurun_out/r2_ensb.json; tail -3 gpurun_out/r2_ensb.err
python bench.py --workload ftr-c2-b128 --no-cpu-baseline > gpurun_out/r2_ftr.json 2> gpurun_out/r2_ftr.err; tail -c 1500 gpurun_out/r2_ftr.json; tail -3 gpurun_out/r2_ftr.err
QPIR_FTR_FUSE=0 python tools/sweep.py ftr-c2-b128 >> gpurun_out/r2_ab.log 2>&1; tail -1 gpurun_out/r2_ab.log
timeout 900 python -m pytest tests -m "gpu and slow" -x -q -s -p no:cacheprovider -k "c4_batch" --durations=0 > gpurun_out/r2_slow.log 2>&1; echo "slow rc=$?"
tail -8 gpurun_out/r2_slow.log
