#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
for c in config1 config3 config5; do echo "== $c"; PROBE_CFG=$c timeout 600 python tools/warp_phases.py 2>&1 | grep -v "^\s*$" | tail -12; done
MCG_PROFILE_BUILD=1 T0=1 T1=2 timeout 600 python tools/prof_c5.py 2>&1 | tail -30
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_warp -s 3 -c 1 \
    -o gpurun_out/c3_warp python tools/prof_warp.py > gpurun_out/ncu_c3w.log 2>&1; echo "ncu c3 rc=$?"
T0=100 T1=103 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_warp -s 1 -c 1 \
    -o gpurun_out/c5_warp python tools/prof_c5.py > gpurun_out/ncu_c5w.log 2>&1; echo "ncu c5 rc=$?"
ls -la gpurun_out
