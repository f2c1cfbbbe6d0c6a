# ncu --set full of one launch each of the non-sweep hot kernels (lines, line factor, coarse V-cycle,
# residual/restriction, cycle update, prep, SpMV, MGS) of a cfg4 solve
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
SPP_NO_GRAPH=1 $CMD > gpurun_out/plain.log 2>&1 && \
SPP_NO_GRAPH=1 timeout 1500 ncu --set full --clock-control none -k regex:'k_lines_tma|k_line_factor_scan|k_coarse_vcycle|k_resid_restrict|k_cycle_update|k_gs_prep|k_spmv|k_mgs' -c 8 -o gpurun_out/prof_others $CMD > gpurun_out/ncu_others.log 2>&1
echo done
