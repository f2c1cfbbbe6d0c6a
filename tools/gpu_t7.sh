mkdir -p gpurun_out
bash tools/ab2.sh
cp tools/ablibs/b_new.so paper_2108_13468_b200/lib/libspp.so
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_new.log 2>&1; tail -2 gpurun_out/gpu_tests_new.log
bash tools/gpu_stress.sh
