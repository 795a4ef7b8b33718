#!/usr/bin/env bash
# One GPU session: bench line, ncu launch list of the same command, one full
# ncu capture of the persistent batch kernel (k_batch), all into gpurun_out/.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 3000 gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other \
    > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_batch -s 20 -c 1 \
    -o gpurun_out/batch_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other \
    > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
