set -x
cd $GRAFT_REPO_ROOT
export CUDA_LAUNCH_BLOCKING=1
for f in 0 1; do for c in "700 33 1" "3001 200 64" "70000 16 9"; do
  QPIR_FTR_FUSE=$f timeout 60 python tools/gpu/ftr_debug.py $c 2>&1 | tail -3
done; done
QPIR_FTR_FUSE=1 QPIR_MMA_MT=1 timeout 60 python tools/gpu/ftr_debug.py 700 33 1 2>&1 | tail -3
unset CUDA_LAUNCH_BLOCKING
for i in 1 2; do
QPIR_LIB=$PWD/paper_2510_03631_b200/libqpir_r1.so python tools/sweep.py c2 -- --steps 2000 --warmup 20
python tools/sweep.py c2 QPIR_GEMV_PF=0,4,8,16 -- --steps 2000 --warmup 20
done > gpurun_out/r3_ab.log 2>&1
QPIR_LIB=$PWD/paper_2510_03631_b200/libqpir_r1.so python tools/sweep.py ens-c2 >> gpurun_out/r3_ab.log 2>&1
python tools/sweep.py ens-c2 >> gpurun_out/r3_ab.log 2>&1
cat gpurun_out/r3_ab.log
QPIR_ENS_TC=1 python bench.py --workload ens-c2-b128 --no-cpu-baseline > gpurun_out/r3_ensb.json 2> gpurun_out/r3_ensb.err; tail -c 2500 gpurun_out/r3_ensb.json; tail -3 gpurun_out/r3_ensb.err
QPIR_FTR_FUSE=0 python tools/sweep.py ftr-c2-b128 2>&1 | tail -2
