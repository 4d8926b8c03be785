set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; free -g | head -2; nproc
python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/r1_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r1_tests.log
python tools/sweep.py c2 QPIR_GEMV_L2PF=0,1 -- --steps 2000 --warmup 20 > gpurun_out/r1_sweep.log 2>&1
python tools/sweep.py ens-c2 QPIR_ENS_PDL=1,0 >> gpurun_out/r1_sweep.log 2>&1
cat gpurun_out/r1_sweep.log
timeout 1500 python -m pytest tests -m "gpu and slow" -x -q -p no:cacheprovider -k "c4_batch or c5_hint" > gpurun_out/r1_slow.log 2>&1; echo "slow rc=$?"
tail -5 gpurun_out/r1_slow.log
