#!/usr/bin/env bash
# FTR (fused 2-limb split) vs the tcgen05 engine's K-lockstep / drift / split knobs.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2ftrls; mkdir -p $O
run() {
  env "$@" timeout 300 python bench.py --workload ftr-c2-b128 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > $O/b.json 2>/dev/null
  python -c "import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print('$*', d['ms_per_step'], d['roofline']['frac'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
}
run QPIR_X=0
run QPIR_MMA_LOCKSTEP=0
run QPIR_MMA_LOCKSTEP=8
run QPIR_MMA_LOCKSTEP=32
run QPIR_MMA_DRIFT=2
run QPIR_MMA_DRIFT=4
run QPIR_MMA_LOCKSTEP=0 QPIR_MMA_SPLIT=12
run QPIR_MMA_SPLIT=12
run QPIR_MMA_SPLIT=4
run QPIR_X=0
