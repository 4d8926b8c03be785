cd $GRAFT_REPO_ROOT
j() { python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'])"; }
for dbg in 0 4 2 6 7; do echo -n "dbg $dbg: "; QPIR_ENS_TS_DBG=$dbg timeout 200 python bench.py --workload ens-c2-b128 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | j; done
