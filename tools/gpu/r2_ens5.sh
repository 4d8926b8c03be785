#!/usr/bin/env bash
timeout 300 python -m pytest tests/test_gpu_ens.py -q -x -k "batch_matches or extreme or ragged" -p no:cacheprovider 2>&1 | tail -1
cd $GRAFT_REPO_ROOT
j() { python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'])"; }
for cfg in 0 1 2 3; do for sp in 0; do
echo -n "cfg $cfg split $sp: "; QPIR_MMA_SPLIT=$sp QPIR_ENS_TS_CFG=$cfg timeout 200 python bench.py --workload ens-c2-b128 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | j
done; done
