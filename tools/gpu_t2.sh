mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --profile-all > gpurun_out/quick.log 2>&1
timeout 300 python bench.py --config cfg3 --no-cpu-baseline --no-e2e > gpurun_out/cfg3.log 2>&1
timeout 300 python bench.py --config cfg2 --no-cpu-baseline --no-e2e > gpurun_out/cfg2.log 2>&1
cp tools/explibs/prof/libspp.so paper_2108_13468_b200/lib/libspp.so
SPP_WAVE_PROF_N=2047 SPP_WAVE_PROF_HIT=1 SPP_WAVE_TL=1 timeout 300 python tools/wave_prof.py > gpurun_out/prof_mii.txt 2>&1
echo done
