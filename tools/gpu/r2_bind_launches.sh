#!/usr/bin/env bash
# Launch list (gpu__time_duration per kernel) of one bind-c2 step.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2bl; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"mldsa|pack_bind" --csv --log-file $O/launches_bind-c2.csv \
    python bench.py --workload bind-c2 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py launches $O/launches_bind-c2.csv $O/r02_launches_bind-c2.md > /dev/null 2>&1; echo "sum rc=$?"
