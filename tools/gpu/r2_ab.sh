#!/usr/bin/env bash
# Same-box A/B: round-1 build vs current (C2 / ENS / FTR variants).  Create the
# round-1 tree first: git worktree add ab_r01 6a560f7 && (cd ab_r01 && python paper_2510_03631_b200/build.py)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2ab; mkdir -p $O
j() { python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'],d['value'],d.get('roofline',{}).get('frac'),d['clocks']['sm_mhz'],d['clocks']['reasons'])"; }
for i in 1 2; do
  echo -n "r01 c2: "; (cd ab_r01 && timeout 120 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null) | j
  echo -n "cur c2: "; timeout 120 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | j
  echo -n "cur c2 pdl0: "; QPIR_GEMV_PDL=0 timeout 120 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | j
done
for w in ens-c2 oop-c2 ftr-c2-b128 ens-c2-b128; do
  echo -n "r01 $w: "; (cd ab_r01 && timeout 200 python bench.py --workload $w --no-cpu-baseline --no-e2e 2>/dev/null) | j
  echo -n "cur $w: "; timeout 200 python bench.py --workload $w --no-cpu-baseline --no-e2e 2>/dev/null | j
done
echo -n "cur ftr fuse0: "; QPIR_FTR_FUSE=0 timeout 200 python bench.py --workload ftr-c2-b128 --no-cpu-baseline --no-e2e 2>/dev/null | j
# launch lists
for w in ftr-c2-b128 ens-c2-b128; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file $O/launches_$w.csv \
    python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
QPIR_FTR_FUSE=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file $O/launches_ftr_fuse0.csv \
    python bench.py --workload ftr-c2-b128 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
(cd ab_r01 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv --log-file ../$O/launches_c2_r01.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1)
ncu --set full --clock-control none --import-source on -k regex:"qpir_ens_mma" -s 2 -c 1 -o $O/ens_mma python bench.py --workload ens-c2-b128 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
