# A/B: bench with env VAR=1 vs default (per-class profile + bench line each), output gpurun_out/ab.log
mkdir -p gpurun_out
for v in "" "$1"; do
  echo "=== env $v" >> gpurun_out/ab.log
  env $v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --profile-all >> gpurun_out/ab.log 2>&1
done
echo done
