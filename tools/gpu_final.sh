#!/usr/bin/env bash
# End-of-round check: GPU suite, smoke, phase breakdowns, bench + reference arm.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_final.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in config3 config5; do echo "== $c"; PROBE_CFG=$c timeout 600 python tools/warp_phases.py 2>&1 | grep -E "window|k_warp phase"; done > gpurun_out/phases_final.txt
bash tools/gpu_session_r02.sh > gpurun_out/session_final.log 2>&1; tail -5 gpurun_out/session_final.log
