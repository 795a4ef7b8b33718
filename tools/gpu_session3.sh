#!/usr/bin/env bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_random.py -x -q -m gpu > gpurun_out/pytest3.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest3.log
timeout 600 python tools/busyring_time.py > gpurun_out/busyring.json 2> gpurun_out/busyring.err; echo "busy rc=$?"; cat gpurun_out/busyring.json; tail -3 gpurun_out/busyring.err
PROBE_T=1000,3000,10000,12000 timeout 600 python tools/phase_probe.py > gpurun_out/phase_c3.txt 2>&1; cat gpurun_out/phase_c3.txt
PROBE_N=100000 PROBE_DEND=large PROBE_T=100,200 timeout 900 python tools/phase_probe.py > gpurun_out/phase_c5.txt 2>&1; cat gpurun_out/phase_c5.txt
