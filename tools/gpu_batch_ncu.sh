# Batched 1D: plain run, then the ncu launch list of the same command and one full capture of
# the solve kernel (each ncu pass only after the plain run exited 0).
mkdir -p gpurun_out
CMD="python bench.py --config cfg1-batch --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/batch_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/batch_launches.csv $CMD > gpurun_out/batch_ncu.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_solve1d_batch -s 0 -c 1 -o gpurun_out/prof_batch1d $CMD > gpurun_out/batch_ncu_full.log 2>&1
echo done
