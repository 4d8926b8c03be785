cd $GRAFT_REPO_ROOT
cat > /tmp/gdbcmds <<'G'
set cuda api_failures ignore
set pagination off
run
p a
p/x a
info cuda warps
quit
G
QPIR_MMA_MT=2 QPIR_FTR_FUSE=0 timeout 300 cuda-gdb -batch -x /tmp/gdbcmds --args python tools/gpu/ftr_debug.py 700 33 1 > gpurun_out/r7_gdb.log 2>&1
grep -v "New Thread\|exited\]" gpurun_out/r7_gdb.log | tail -40
cat > /tmp/t.py <<'P'
import ctypes, paper_2510_03631_b200 as P
P._lib.QPIR_FLAG_STABLE_INPUTS
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
P
