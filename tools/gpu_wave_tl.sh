mkdir -p gpurun_out
./tools/ubench/lat > gpurun_out/lat.txt 2>&1
cp tools/explibs/prof/libspp.so paper_2108_13468_b200/lib/libspp.so
SPP_WAVE_PROF_N=4095 SPP_WAVE_PROF_HIT=1 SPP_WAVE_TL=1 timeout 300 python tools/wave_prof.py > gpurun_out/prof_mii.txt 2>&1
SPP_WAVE_PROF_N=4095 SPP_WAVE_PROF_HIT=3 SPP_WAVE_TL=1 timeout 300 python tools/wave_prof.py > gpurun_out/prof_mii3.txt 2>&1
SPP_WAVE_PROF_N=2048 SPP_WAVE_PROF_HIT=3 SPP_WAVE_TL=1 timeout 300 python tools/wave_prof.py > gpurun_out/prof_l0.txt 2>&1
SPP_WAVE_PROF_N=256 SPP_WAVE_PROF_HIT=3 SPP_WAVE_TL=1 timeout 300 python tools/wave_prof.py > gpurun_out/prof_l3.txt 2>&1
echo done
