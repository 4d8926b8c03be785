#!/usr/bin/env bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2ftr; mkdir -p $O
j() { python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d.get('roofline',{}).get('frac'),d['clocks']['sm_mhz'],d['clocks']['reasons'], d.get('e2e',{}) and d['e2e'].get('ms_per_step'))"; }
timeout 900 python -m pytest tests/test_gpu_ftr.py tests/test_gpu_parity.py tests/test_gpu_ens.py -q -x -k "not slow and not c4_batch_sampled and not c5_hint" -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for i in 1 2; do
echo -n "c2: "; timeout 120 python bench.py --no-cpu-baseline 2>/dev/null | j
echo -n "ftr fuse1: "; timeout 200 python bench.py --workload ftr-c2-b128 --no-cpu-baseline --no-e2e 2>/dev/null | j
echo -n "ftr fuse0: "; QPIR_FTR_FUSE=0 timeout 200 python bench.py --workload ftr-c2-b128 --no-cpu-baseline --no-e2e 2>/dev/null | j
done
echo -n "ens-c2: "; timeout 200 python bench.py --workload ens-c2 --no-cpu-baseline --no-e2e 2>/dev/null | j
echo -n "oop-c2: "; timeout 200 python bench.py --workload oop-c2 --no-cpu-baseline --no-e2e 2>/dev/null | j
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file $O/launches_ftr.csv \
    python bench.py --workload ftr-c2-b128 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
