mkdir -p gpurun_out
cp tools/explibs/cprof/libspp.so paper_2108_13468_b200/lib/libspp.so
timeout 120 python bench.py --config cfg2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep "\[coarse\]" | head -4
bash tools/ab2.sh
cp tools/ablibs/b_czf.so paper_2108_13468_b200/lib/libspp.so
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_czf.log 2>&1; tail -2 gpurun_out/gpu_tests_czf.log
