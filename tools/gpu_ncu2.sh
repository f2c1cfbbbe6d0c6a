# full ncu capture (source-level sampling) of the first k_wave launches of a cfg4 solve
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
SPP_NO_GRAPH=1 $CMD > gpurun_out/plain.log 2>&1 && \
SPP_NO_GRAPH=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 0 -c 2 -o gpurun_out/prof_wave5 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
