#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke4.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke4.log
timeout 600 python tools/warp_ab.py > gpurun_out/ab_c3.txt 2>&1; cat gpurun_out/ab_c3.txt
PROBE_N=100000 PROBE_DEND=large PROBE_T=100,300 timeout 900 python tools/warp_ab.py > gpurun_out/ab_c5.txt 2>&1; cat gpurun_out/ab_c5.txt
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/pytest4.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest4.log
