# Parity tests, then bench variants of the kernel tunables (cfg4), per-class profile to stderr.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
for t in "" "gs_tile_cols=512" "gs_tile_cols=256"; do
  echo "=== SPP_TUNE=$t" >> gpurun_out/tune.log
  SPP_TUNE="$t" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --profile-all >> gpurun_out/tune.log 2>&1
done
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1
echo done
