#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
for g in 1 2 3 4 5; do echo "== G=$g"; MCG_WARP_G=$g PROBE_T=1000,3000,10000,12000 timeout 600 python tools/warp_phases.py 2>&1 | grep -E "window|engine:"; done
for g in 2 3 5; do echo "== c5 G=$g"; MCG_WARP_G=$g PROBE_CFG=config5 PROBE_T=100,200 timeout 600 python tools/warp_phases.py 2>&1 | grep -E "window|engine:"; done
