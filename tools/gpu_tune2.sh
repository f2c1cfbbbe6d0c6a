# bench variants of SPP_TUNE given as arguments (cfg4), per-class profile
mkdir -p gpurun_out
for t in "$@"; do
  echo "=== SPP_TUNE=$t" >> gpurun_out/tune2.log
  SPP_TUNE="$t" timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --profile-all >> gpurun_out/tune2.log 2>&1
done
echo done
