#!/usr/bin/env bash
# Signer iteration: bind tests, bind-c2 bench, one ncu capture of mldsa_sign_kernel.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2sign; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_bind.py -q -x -p no:cacheprovider > $O/pytest_bind.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_bind.log
for i in 1 2; do timeout 300 python bench.py --workload bind-c2 --steps 4 --warmup 3 --no-cpu-baseline > $O/bench_bind_$i.json 2>$O/bench_bind_$i.err; echo "bench rc=$?"; python -c "import json;d=json.load(open('$O/bench_bind_$i.json'));print(d['ms_per_step'],d['roofline']['frac'],d['clocks'])"; done
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mldsa_sign -s 1 -c 1 \
   -o $O/sign2 python tools/gpu/sign_probe.py > $O/ncu2.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py full $O/sign2.ncu-rep $O/r02_mldsa_sign2_ncu_full.md > /dev/null 2>&1; echo "sum rc=$?"
fi
