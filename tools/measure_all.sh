#!/usr/bin/env bash
# Reproduce the round's measurements on a B200 (run from the repo root, e.g.
#   gpurun --timeout 3000 -- 'bash tools/measure_all.sh'
# ).  Bench JSON lines -> gpurun_out/final/, ncu summaries + DRAM traffic ->
# gpurun_out/ (copy what should be judged into profiles/).
set -u
mkdir -p gpurun_out/final
python -m pytest tests -q -m gpu 2>&1 | tail -1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err
for w in c1 c2 c3 c4-64 c4-256 c5 ens-c2 ens-c2-b128 ftr-c2-b128 oop-c2; do
  python bench.py --workload "$w" > "gpurun_out/final/bench_$w.json" 2> "gpurun_out/final/bench_$w.err"
done
python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
# one `ncu --set full` capture of each workload's dominant kernel (serialised, cold)
for w in c1 c2 c3 c4-64 c4-256 c5 ftr-c2-b128 ens-c2 ens-c2-b128 oop-c2; do
  ncu --set full --clock-control none -k regex:"gemv_u8|mma_u8|ens_scan" -s 3 -c 1 \
      -o "/tmp/prof_$w" python bench.py --workload "$w" --steps 5 --warmup 3 --graph 0 \
      --no-cpu-baseline --no-e2e > /dev/null 2>&1
  python tools/ncu_summary.py full "/tmp/prof_$w.ncu-rep" "gpurun_out/r01_final_${w}_ncu_full.md" \
      --traffic "gpurun_out/traffic_$w.json" > /dev/null 2>&1
  rm -f "/tmp/prof_$w.ncu-rep"
done
# launch list of the default bench step (gpu__time_duration per kernel)
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemv|limb|mma|pack|ens|modp|expand" \
    -c 40 --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_c2.csv gpurun_out/launches_c2.md > /dev/null
