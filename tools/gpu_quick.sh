# Parity tests + one bench line with the per-class profile (cfg4) + launch list of the k_wave sweeps.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
tail -1 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --profile-all > gpurun_out/quick.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_wave -c 12 --csv --log-file gpurun_out/wave_launches.csv $CMD > gpurun_out/ncu_q.log 2>&1
echo done
