# A/B of tools/ablibs/*.so (cfg4 / cfg3 / cfg2), then the GPU suite with the candidate library $1
mkdir -p gpurun_out
bash tools/ab2.sh
cp tools/ablibs/$1 paper_2108_13468_b200/lib/libspp.so
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_ab.log 2>&1; tail -2 gpurun_out/gpu_tests_ab.log
