#!/usr/bin/env bash
# Round-2 ncu evidence: one `ncu --set full` capture of each workload's dominant
# kernel (summarised to profiles/r02_<w>_ncu_full.md + DRAM traffic json) and the
timeout 900 python -m pytest tests/test_gpu_bind.py tests/test_gpu_ens.py -q -x -p no:cacheprovider > gpurun_out/r2p_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2p_pytest.log
# launch lists (gpu__time_duration per kernel) of the default bench and the NEXT rows.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2p; mkdir -p $O
for w in c2 c4-64 c4-256 c5 ftr-c2-b128 ens-c2 ens-c2-b128 oop-c2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemv_u8|mma_u8|ens_scan|qpir_ens_mma" -s 3 -c 1 \
      -o "/tmp/prof_$w" python bench.py --workload "$w" --steps 5 --warmup 3 --graph 0 \
      --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "$w rc=$?"
  python tools/ncu_summary.py full "/tmp/prof_$w.ncu-rep" "$O/r02_${w}_ncu_full.md" --traffic "$O/traffic_$w.json" > /dev/null 2>&1
done
for w in c2 c4-64 ftr-c2-b128 ens-c2-b128 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"gemv|mma_u8|limb_split|modp_fixup|ens_share|ens_mma|ens_scan|expand_A" -c 40 --csv --log-file $O/launches_$w.csv \
      python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python tools/ncu_summary.py launches $O/launches_$w.csv $O/r02_launches_$w.md > /dev/null 2>&1
  echo "launches $w rc=$?"
done
ls $O; du -sh $O
