mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/list_cfg4.csv $CMD > gpurun_out/ncu4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/list_cfg3.csv $CMD --config cfg3 > gpurun_out/ncu3.log 2>&1
echo done
