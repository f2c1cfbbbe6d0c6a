mkdir -p gpurun_out
for d in 0 2 4 6 24 30; do
  echo "=== SPP_WAVE_DBG=$d" >> gpurun_out/dbg.log
  SPP_WAVE_DBG=$d timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e --profile-all 2>&1 | grep -E "mg_sweep|sweep_I|ms_per" | cut -c1-140 >> gpurun_out/dbg.log
done
