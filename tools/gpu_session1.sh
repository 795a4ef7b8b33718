set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_configs.py tests/test_gpu_dropin.py -x -q -m gpu --durations=20 > gpurun_out/pytest_configs.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_configs.log
python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"; cat gpurun_out/ref.json
python tools/prof_c5.py > gpurun_out/c5.log 2>&1; cat gpurun_out/c5.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch -s 1 -c 1 -o gpurun_out/c5_full python tools/prof_c5.py > gpurun_out/ncu_c5.log 2>&1; echo "ncu rc=$?"; tail -5 gpurun_out/ncu_c5.log
