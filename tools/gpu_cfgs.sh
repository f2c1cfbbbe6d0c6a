# The other BASELINE configs on one GPU (time-to-solution lines)
mkdir -p gpurun_out
for e in 1e-10 1e-8 1e-6; do timeout 900 python bench.py --config cfg5 --eps $e --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfgs_cfg5_$e.log 2>&1; done
timeout 600 python bench.py --config cfg3 --no-cpu-baseline --no-e2e > gpurun_out/cfgs_cfg3.log 2>&1
timeout 600 python bench.py --config cfg2 --no-cpu-baseline --no-e2e > gpurun_out/cfgs_cfg2.log 2>&1
timeout 900 python bench.py --config cfg5-sweep --steps 1 --warmup 1 > gpurun_out/cfgs_sweep.log 2>&1
timeout 600 python bench.py --config cfg1-batch > gpurun_out/cfgs_batch.log 2>&1
echo done
