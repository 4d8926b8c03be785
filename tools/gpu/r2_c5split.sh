#!/usr/bin/env bash
# C5 hint: K-split count vs time, sustained clock and DRAM bytes (A' chunk L2-resident
# when the split's K range of A' fits in L2)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c5; mkdir -p $O
j() { python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'],d['clocks'].get('power_w_median'),d['clocks']['reasons'])"; }
for sp in 0 8 16 24 32; do
  echo -n "split $sp: "; QPIR_MMA_SPLIT=$sp timeout 300 python bench.py --workload c5 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | j
done
for sp in 0 16 24; do
  QPIR_MMA_SPLIT=$sp timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:mma_u8 -s 3 -c 1 --csv --log-file $O/c5_split$sp.csv python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "ncu split $sp"; grep -E "dram__bytes|gpu__time|lts__t_bytes" $O/c5_split$sp.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
