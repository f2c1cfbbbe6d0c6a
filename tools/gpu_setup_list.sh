# launch list (ncu, duration only) of the setup kernels of one cfg4 step
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_line_factor|k_coef|k_validate|k_ycoef|k_level_rho|k_level0|k_pack|k_rhs|k_scale' -c 60 --csv --log-file gpurun_out/setup_launches.csv $CMD > gpurun_out/ncu_s.log 2>&1
echo done
