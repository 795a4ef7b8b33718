#!/usr/bin/env bash
# quick loop: phase timing at config 3 (+ optional extra), then the given pytest selection
set -u
mkdir -p gpurun_out
PROBE_T=1000,3000,10000,12000 timeout 600 python tools/warp_phases.py 2>&1 | grep -E "window|engine:|k_warp phase" | tail -9
if [ -n "${EXTRA:-}" ]; then eval "$EXTRA"; fi
if [ -n "${TESTS:-}" ]; then timeout 1800 python -m pytest -x -q $TESTS 2>&1 | tail -4; fi
