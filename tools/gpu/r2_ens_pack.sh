#!/usr/bin/env bash
# ENS share packing (transposed through smem): ENS / OOP tests, ens-c2-b128 bench, launch list.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2ep; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ens.py tests/test_gpu_oop.py tests/test_gpu_bind.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for i in 1 2; do
  timeout 300 python bench.py --workload ens-c2-b128 --steps 100 --warmup 5 --no-cpu-baseline > $O/b$i.json 2>/dev/null
  python -c "import json;d=json.loads(open('$O/b$i.json').read().strip().splitlines()[-1]);print('ens-b128', d['ms_per_step'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"ens_share|ens_mma" -c 40 --csv --log-file $O/launches.csv \
    python bench.py --workload ens-c2-b128 --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py launches $O/launches.csv $O/r02_launches_ens-c2-b128.md > /dev/null 2>&1; cat $O/r02_launches_ens-c2-b128.md
