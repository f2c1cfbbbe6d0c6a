# full ncu capture (source-level sampling) of one k_lines launch and one k_coarse_vcycle launch
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
SPP_NO_GRAPH=1 $CMD > gpurun_out/plain.log 2>&1 && \
SPP_NO_GRAPH=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_lines' -s 0 -c 1 -o gpurun_out/prof_lines $CMD > gpurun_out/ncu_lines.log 2>&1
echo done
