#!/usr/bin/env bash
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_ens.py -q -x -k "batch_matches or extreme or ragged or mutation or bruteforce" -p no:cacheprovider 2>&1 | tail -3
j() { python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'])"; }
for i in 1 2; do for pr in 1 0; do
echo -n "pair $pr: "; QPIR_ENS_PAIR=$pr timeout 200 python bench.py --workload ens-c2-b128 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | j
done; done
