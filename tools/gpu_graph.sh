mkdir -p gpurun_out
SPP_DEBUG_GRAPH=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g1.log 2>&1
SPP_NO_GRAPH=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g0.log 2>&1
echo done
