# Parity check then one full ncu capture of selected k_gs_rows launches of a cfg4 solve
mkdir -p gpurun_out
#timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
tail -3 gpurun_out/gpu_tests.log
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 0 -c 6 -o gpurun_out/prof_wave4 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
