#!/usr/bin/env bash
# Round-2 measurement session: bench line (+ reference arm), launch list of the
# same command, ncu captures of the stepping kernels, the config-1 timing.
set -u
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other \
    > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_warp -s 20 -c 1 \
    -o gpurun_out/warp_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other \
    > gpurun_out/ncu_full.log 2>&1; echo "ncu k_warp rc=$?"
T0=100 T1=103 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_warp -s 1 -c 1 \
    -o gpurun_out/c5_warp python tools/prof_c5.py > gpurun_out/ncu_c5w.log 2>&1; echo "ncu c5 rc=$?"
T_END=8000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_point -s 0 -c 1 \
    -o gpurun_out/pt python tools/prof_point.py > gpurun_out/ncu_pt.log 2>&1; echo "ncu k_point rc=$?"
timeout 600 python tools/config1_time.py > gpurun_out/config1.txt 2>&1; tail -4 gpurun_out/config1.txt
timeout 600 python tools/setup_time.py > gpurun_out/setup.txt 2>&1; tail -2 gpurun_out/setup.txt
ls -la gpurun_out
