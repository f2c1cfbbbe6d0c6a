mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_restart.py -q -x -p no:cacheprovider > gpurun_out/gpu_restart.log 2>&1; tail -3 gpurun_out/gpu_restart.log
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/quick.log 2>&1; grep -o 'ms_per_step": [0-9.]*' gpurun_out/quick.log
bash tools/gpu_stress.sh
