set -x
cd $GRAFT_REPO_ROOT
export QPIR_DEBUG_SYNC=1
for mt in 2 1; do for f in 0 1; do
  QPIR_MMA_MT=$mt QPIR_FTR_FUSE=$f timeout 60 python tools/gpu/ftr_debug.py 700 33 1 2>&1 | tail -1
done; done
python - <<'PY'
import numpy as np, synth, paper_2510_03631_b200 as P
from oracle import oracle as O
for (nc, nch, d) in [(700, 1, 33), (1200, 6, 30)]:
    rec = synth.records_np(1, nc * nch, d, nch); D = O.pack(rec, nc, nch, d, nc)
    Q = synth.uniform_u32_np(5, (3, nc))
    try:
        with P.PirServer(nc, nch, d, records=rec) as s:
            print("LWE batch", nc, nch, d, (P.u32(s.answer_batch(Q)) == O.answer_batch(D, Q)).all(), flush=True)
    except Exception as e:
        print("LWE batch", nc, nch, d, "ERR", e, flush=True)
PY
