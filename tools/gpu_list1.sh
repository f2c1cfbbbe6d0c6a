# full launch list (ncu, duration only) of ONE cfg4 solve (setup + solve, no warm-up)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/list1.csv $CMD > gpurun_out/ncu_l1.log 2>&1
echo done
