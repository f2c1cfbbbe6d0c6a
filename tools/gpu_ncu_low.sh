# ncu --set full of the V-cycle's HBM-bound level kernels (restriction of the pre-smoothing
# residual, prolongation + post-smoothing rhs, cycle update) on one cfg4 solve (host-driven loop)
O=gpurun_out/ncu_low
mkdir -p $O
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
SPP_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_restrict_low|k_gs_prep|k_cycle_update" -c 14 -o $O/prof_low $CMD > $O/ncu.log 2>&1
echo "ncu rc=$?"
