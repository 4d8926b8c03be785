#!/usr/bin/env bash
# FTR mod-p fixup (Barrett, 32-bit index math): FTR / batch parity tests, ftr bench, launch list.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2fx; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ftr.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "ftr or modp or prime or batch" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest.log
for i in 1 2; do
  timeout 300 python bench.py --workload ftr-c2-b128 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > $O/b$i.json 2>/dev/null
  python -c "import json;d=json.loads(open('$O/b$i.json').read().strip().splitlines()[-1]);print('ftr', d['ms_per_step'], d['roofline']['frac'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mma_u8|modp_fixup" -c 20 --csv --log-file $O/launches.csv \
    python bench.py --workload ftr-c2-b128 --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py launches $O/launches.csv $O/r02_launches_ftr-c2-b128.md > /dev/null 2>&1; cat $O/r02_launches_ftr-c2-b128.md
