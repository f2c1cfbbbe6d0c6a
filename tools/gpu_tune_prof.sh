bash tools/gpu_tune.sh
SPP_WAVE_DBG=64 SPP_WAVE_PROF_DUMP=1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep wave-prof > gpurun_out/waveprof.log
