# Batched 1D (NEXT-3): GPU tests of the batch + 1D paths, then the cfg1-batch bench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batch1d.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "batch or cfg1 or table2" > gpurun_out/batch_tests.log 2>&1
timeout 600 python bench.py --config cfg1-batch --no-cpu-baseline > gpurun_out/batch_bench.log 2>&1
timeout 600 python bench.py --config cfg1-batch --batch 2048 --no-cpu-baseline --no-e2e >> gpurun_out/batch_bench.log 2>&1
echo done
