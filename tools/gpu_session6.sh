#!/usr/bin/env bash
# Round-2 re-entry session: GPU tests, bench line, launch list, config-5 capture.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest6.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest6.log
timeout 900 python bench.py > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench6.json
timeout 600 python tools/warp_ab.py 2>&1 | tail -3
PROBE_N=100000 PROBE_DEND=large PROBE_T=100,300 timeout 900 python tools/warp_ab.py 2>&1 | tail -3
timeout 900 python tools/config1_time.py 2>&1 | tail -5
T0=100 T1=103 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 3 -c 1 \
    -o gpurun_out/c5_full python tools/prof_c5.py > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
ls -la gpurun_out
