#!/usr/bin/env bash
# End-of-round-2 measurement: GPU suite, smoke, bench + reference arm, launch
# list, ncu captures (k_warp config 3 / config 5, k_point, k_batch busyring),
# config-1 and setup timings.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/gpu_session_r02.sh
T_END=60 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 0 -c 1 \
    -o gpurun_out/busy_final python tools/prof_busyring.py > gpurun_out/ncu_busy_final.log 2>&1; echo "busy rc=$?"
MCG_PHASE_TIMING=1 MCG_VERBOSE=1 T_END=200 timeout 300 python tools/prof_busyring.py > gpurun_out/busy_phase_final.txt 2>&1
