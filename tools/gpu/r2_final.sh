#!/usr/bin/env bash
# Round-2 validation: full GPU suite, smoke, every bench line, launch lists.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2f; mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider --durations=10 > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
for w in c2 c1 c4-64 c4-256 c5 ens-c2 ens-c2-b128 ftr-c2-b128 oop-c2 bind-c2 bind-c2-unsigned; do
  timeout 400 python bench.py --workload "$w" > "$O/bench_$w.json" 2> "$O/bench_$w.err"
  echo "$w rc=$?"
done
timeout 900 python bench.py --workload c3 > $O/bench_c3.json 2> $O/bench_c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
for w in c2 c4-64 ftr-c2-b128 ens-c2-b128 c5 bind-c2 bind-c2-unsigned; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:"gemv|mma_u8|limb_split|modp_fixup|ens_share|ens_mma|ens_scan|expand_A|pack_bind|mldsa" -c 40 --csv --log-file $O/launches_$w.csv \
      python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python tools/ncu_summary.py launches $O/launches_$w.csv $O/r02_launches_$w.md > /dev/null 2>&1
  echo "launches $w rc=$?"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"pack_bind" -s 3 -c 1 -o /tmp/prof_bind python bench.py --workload bind-c2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py full /tmp/prof_bind.ncu-rep $O/r02_bind-c2_ncu_full.md --traffic $O/traffic_bind-c2.json > /dev/null 2>&1
du -sh $O
