#!/usr/bin/env bash
for g in 2 3 4 5; do echo "== G=$g"; MCG_WARP_G=$g PROBE_T=3000,10000,12000 timeout 600 python tools/warp_phases.py 2>&1 | grep -E "window|engine: k_warp"; done
for g in 3 5; do echo "== n4000 G=$g"; MCG_WARP_G=$g PROBE_CFG=n4000 PROBE_T=3000,10000,12000 timeout 600 python tools/warp_phases.py 2>&1 | grep -E "window|engine: k_warp"; done
