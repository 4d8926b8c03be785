#!/usr/bin/env bash
# Signer iteration: bind tests, bind-c2 bench x2, ncu capture + per-line summary.
cd $GRAFT_REPO_ROOT
NCU=0 bash tools/gpu/r2_sign_iter.sh
bash tools/gpu/r2_sign_ncu_only.sh
python tools/ncu_lines.py gpurun_out/r2sign/sign3.ncu-rep 40 > gpurun_out/r2sign/lines.txt 2>&1
