#!/usr/bin/env bash
# Round-2 baseline session: full GPU parity suite, bench line, config-5 ncu capture.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 4000 gpurun_out/bench.json
timeout 600 python tools/prof_c5.py > gpurun_out/c5.log 2>&1; cat gpurun_out/c5.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 1 -c 1 -o gpurun_out/c5_full python tools/prof_c5.py > gpurun_out/ncu_c5.log 2>&1; echo "ncu rc=$?"; tail -5 gpurun_out/ncu_c5.log
ls -la gpurun_out
