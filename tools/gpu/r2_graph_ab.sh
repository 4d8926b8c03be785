#!/usr/bin/env bash
# Stream launches vs one CUDA graph of the K timed steps, per workload.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2g; mkdir -p $O
for w in ftr-c2-b128 ens-c2-b128 c4-64 ens-c2 oop-c2 c2; do
  for g in 0 1; do
    timeout 300 python bench.py --workload $w --steps 200 --warmup 5 --graph $g --no-cpu-baseline --no-e2e > $O/b.json 2>$O/b.err
    python -c "import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print('$w graph=$g', d['ms_per_step'], d['roofline']['frac'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'), d.get('gpu_launches'))" || tail -3 $O/b.err
  done
done
