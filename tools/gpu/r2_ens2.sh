#!/usr/bin/env bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2ens2; mkdir -p $O
j() { python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d.get('roofline',{}).get('frac'),d['clocks']['sm_mhz'],d['clocks']['reasons'], d.get('e2e',{}) and d['e2e'].get('ms_per_step'))"; }
timeout 300 python -m pytest tests/test_gpu_ens.py -q -x -k "batch_matches or extreme or ragged or mutation or bruteforce" -p no:cacheprovider > $O/pytest_ens.log 2>&1; echo "pytest ens rc=$?"; tail -3 $O/pytest_ens.log
for i in 1; do
echo -n "ens128 ts1: "; timeout 200 python bench.py --workload ens-c2-b128 --no-cpu-baseline --no-e2e 2>/dev/null | j
echo -n "ens128 ts0: "; QPIR_ENS_TS=0 timeout 200 python bench.py --workload ens-c2-b128 --no-cpu-baseline --no-e2e 2>/dev/null | j
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"qpir_ens_mma" -s 2 -c 1 -o $O/ens_ts python bench.py --workload ens-c2-b128 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
for i in 1 2; do
echo -n "r01 c2: "; (cd ab_r01 && timeout 120 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null) | j
echo -n "cur c2: "; timeout 120 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | j
done
