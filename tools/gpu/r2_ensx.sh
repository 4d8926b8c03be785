#!/usr/bin/env bash
cd $GRAFT_REPO_ROOT
j() { python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'])"; }
for i in 1 2 3; do echo -n "head: "; timeout 200 python bench.py --workload ens-c2-b128 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | j; done
