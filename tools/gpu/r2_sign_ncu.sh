#!/usr/bin/env bash
# One `ncu --set full` capture of mldsa_sign_kernel (16384 records) with source.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2sign; mkdir -p $O
timeout 300 python tools/gpu/sign_probe.py; echo "probe rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mldsa_sign -s 1 -c 1 \
   -o $O/sign python tools/gpu/sign_probe.py > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py full $O/sign.ncu-rep $O/r02_mldsa_sign_ncu_full.md > /dev/null 2>&1; echo "sum rc=$?"
