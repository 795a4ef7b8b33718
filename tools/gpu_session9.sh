#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
T_END=10600 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_warp -s 108 -c 1 \
    -o gpurun_out/c3_learn python tools/prof_warp.py > gpurun_out/ncu_c3l.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/c3_learn.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c3_learn_src.csv 2>/dev/null
ls -la gpurun_out
