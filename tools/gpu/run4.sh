set -x
cd $GRAFT_REPO_ROOT
export CUDA_LAUNCH_BLOCKING=1
for lib in new r1; do
  if [ $lib = r1 ]; then export QPIR_LIB=$PWD/paper_2510_03631_b200/libqpir_r1.so; fi
  for mt in 2 1; do for gpb in 8 4; do for f in 0 1; do
    echo "lib=$lib mt=$mt gpb=$gpb fuse=$f"
    QPIR_MMA_MT=$mt QPIR_MMA_GPB=$gpb QPIR_FTR_FUSE=$f timeout 60 python tools/gpu/ftr_debug.py 700 33 1 2>&1 | tail -1
  done; done; done
  unset QPIR_LIB
done
QPIR_MMA_MT=2 QPIR_FTR_FUSE=0 timeout 60 python tools/gpu/ftr_debug.py 700 33 64 2>&1 | tail -1
QPIR_MMA_MT=2 QPIR_FTR_FUSE=0 timeout 60 python tools/gpu/ftr_debug.py 5000 300 128 2>&1 | tail -1
unset CUDA_LAUNCH_BLOCKING
python tools/sweep.py c2 QPIR_GEMV_PF=0,4,8,16 -- --steps 2000 --warmup 20 > gpurun_out/r4_ab.log 2>&1
QPIR_LIB=$PWD/paper_2510_03631_b200/libqpir_r1.so python tools/sweep.py c2 -- --steps 2000 --warmup 20 >> gpurun_out/r4_ab.log 2>&1
python tools/sweep.py c2 QPIR_GEMV_PF=8,16 -- --steps 2000 --warmup 20 >> gpurun_out/r4_ab.log 2>&1
cat gpurun_out/r4_ab.log
