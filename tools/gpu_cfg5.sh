# cfg5 (8192^2, 67M unknowns) eps sweep on one GPU: bench lines (no CPU baseline / e2e)
mkdir -p gpurun_out
for e in 1e-6 1e-8 1e-10; do
  timeout 600 python bench.py --config cfg5 --eps $e --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg5_$e.log 2>&1
  tail -1 gpurun_out/cfg5_$e.log | cut -c1-400
done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
