#!/usr/bin/env bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c5h; mkdir -p $O
j() { python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'],d['clocks'].get('power_w_median'),d['clocks']['reasons'])"; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "hint or batch" -p no:cacheprovider 2>&1 | tail -1
for cfg in "0 0" "0 3" "16 0" "16 3" "16 2" "24 3" "12 3"; do set -- $cfg
  echo -n "split $1 hint $2: "; QPIR_MMA_SPLIT=$1 QPIR_MMA_L2HINT=$2 timeout 300 python bench.py --workload c5 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | j
done
for cfg in "0 3" "16 3" "16 2"; do set -- $cfg
  QPIR_MMA_SPLIT=$1 QPIR_MMA_L2HINT=$2 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:mma_u8 -s 3 -c 1 --csv --log-file $O/c5_$1_$2.csv python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "ncu split $1 hint $2"; grep -E "dram__bytes|gpu__time" $O/c5_$1_$2.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
