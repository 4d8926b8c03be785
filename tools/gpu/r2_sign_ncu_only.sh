cd $GRAFT_REPO_ROOT; O=gpurun_out/r2sign; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mldsa_sign -s 1 -c 1 -o $O/sign3 python tools/gpu/sign_probe.py > $O/ncu3.log 2>&1; echo "ncu rc=$?"
