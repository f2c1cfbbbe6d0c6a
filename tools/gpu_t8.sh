mkdir -p gpurun_out
cp tools/ablibs/b_lines.so paper_2108_13468_b200/lib/libspp.so
SPP_DEBUG_LINES=1 timeout 120 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep "line chains" | head -2
bash tools/ab2.sh
cp tools/ablibs/b_lines.so paper_2108_13468_b200/lib/libspp.so
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_lines.log 2>&1; tail -2 gpurun_out/gpu_tests_lines.log
