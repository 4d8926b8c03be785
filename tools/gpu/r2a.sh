cd $GRAFT_REPO_ROOT
for f in 0 1; do QPIR_FTR_FUSE=$f timeout 60 python tools/gpu/ftr_debug.py 700 33 1 2>&1 | tail -1; done
QPIR_FTR_FUSE=1 timeout 60 python tools/gpu/ftr_debug.py 5000 300 128 2>&1 | tail -1
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/r2a_tests.log
