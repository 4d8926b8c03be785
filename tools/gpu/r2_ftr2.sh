#!/usr/bin/env bash
cd $GRAFT_REPO_ROOT
j() { python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'])"; }
timeout 300 python -m pytest tests/test_gpu_ftr.py -q -x -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do
echo -n "fuse1: "; QPIR_FTR_FUSE=1 timeout 200 python bench.py --workload ftr-c2-b128 --no-cpu-baseline --no-e2e 2>/dev/null | j
echo -n "fuse0: "; QPIR_FTR_FUSE=0 timeout 200 python bench.py --workload ftr-c2-b128 --no-cpu-baseline --no-e2e 2>/dev/null | j
done
QPIR_FTR_FUSE=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"mma_u8|modp" -c 6 --csv --log-file gpurun_out/ftr_fuse.csv python bench.py --workload ftr-c2-b128 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > /dev/null 2>&1
grep -E "gpu__time|dram" gpurun_out/ftr_fuse.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | head -12
