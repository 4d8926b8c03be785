#!/usr/bin/env bash
cd $GRAFT_REPO_ROOT
j() { python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'])"; }
timeout 300 python -m pytest tests/test_gpu_ftr.py -q -x -p no:cacheprovider 2>&1 | tail -1
for i in 1 2 3; do echo -n "fuse1: "; timeout 200 python bench.py --workload ftr-c2-b128 --no-cpu-baseline --no-e2e 2>/dev/null | j; done
echo -n "fuse0: "; QPIR_FTR_FUSE=0 timeout 200 python bench.py --workload ftr-c2-b128 --no-cpu-baseline --no-e2e 2>/dev/null | j
