#!/usr/bin/env bash
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_ens.py -q -x -k "batch_matches or extreme or ragged" -p no:cacheprovider 2>&1 | tail -1
j() { python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'])"; }
for i in 1 2; do for shx in 0 1; do
echo -n "shx $shx: "; QPIR_ENS_SHX=$shx timeout 200 python bench.py --workload ens-c2-b128 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | j
done; done
