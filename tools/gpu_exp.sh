# timing experiments: per-k_wave-launch durations (ncu list) of one solve for the given build tag
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
SPP_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_wave -c 7 --csv --log-file gpurun_out/exp_$1.csv $CMD > gpurun_out/exp_$1.log 2>&1
echo done
