#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest5.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest5.log
timeout 600 python tools/warp_ab.py 2>&1 | tail -3
PROBE_N=100000 PROBE_DEND=large PROBE_T=100,300 timeout 900 python tools/warp_ab.py 2>&1 | tail -3
PROBE_N=4000 PROBE_T=500,2500 timeout 900 python tools/warp_ab.py 2>&1 | tail -3
timeout 900 python tools/config1_time.py 2>&1 | tail -5
