#!/usr/bin/env bash
# end-of-round profile refresh: busyring, busyring+STDP, config 2 (k_batch), config 3 (k_warp)
set -u
mkdir -p gpurun_out
T_END=60 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 0 -c 1 \
    -o gpurun_out/busy_s5 python tools/prof_busyring.py > gpurun_out/ncu_busy_s5.log 2>&1; echo "busy rc=$?"
BUSY_STDP=1 T_END=60 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 0 -c 1 \
    -o gpurun_out/busystdp_s5 python tools/prof_busyring.py > gpurun_out/ncu_busystdp_s5.log 2>&1; echo "busy stdp rc=$?"
T_END=1500 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 0 -c 1 \
    -o gpurun_out/cfg2_s5 python tools/prof_config2.py > gpurun_out/ncu_cfg2_s5.log 2>&1; echo "cfg2 rc=$?"
# k_warp captured in the first pass of this script (warp_s5)
false && \
    -o gpurun_out/warp_s5 python tools/prof_warp.py > gpurun_out/ncu_warp_s5.log 2>&1; echo "warp rc=$?"
timeout 300 python tools/busyring_time.py > gpurun_out/busy_time_s5.txt 2>&1; tail -3 gpurun_out/busy_time_s5.txt
