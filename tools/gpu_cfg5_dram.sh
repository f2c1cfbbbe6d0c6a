# cfg5 (8192^2, eps = 1e-10): bench line, then DRAM bytes + duration of the first k_wave launches
mkdir -p gpurun_out
CMD="python bench.py --config cfg5 --eps 1e-10 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
SPP_NO_GRAPH=1 $CMD > gpurun_out/c5_plain.log 2>&1 && \
SPP_NO_GRAPH=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_wave -c 40 --csv --log-file gpurun_out/c5_wave_dram.csv $CMD > gpurun_out/c5_ncu.log 2>&1
timeout 600 python bench.py --config cfg5 --eps 1e-10 --no-cpu-baseline --profile-all > gpurun_out/c5_bench.log 2>&1
echo done
