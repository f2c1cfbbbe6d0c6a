for t in "sweep_warps=2" "sweep_warps=1" "sweep_warps=3" "sweep_warps=4" "sweep_warps=5" "gs_lag=3" "gs_lag=4" "gs_lag=6" "gs_warps=4" "gs_warps=3" "gs_max_halo=0"; do
  r=$(SPP_TUNE=$t timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-all 2>&1 | grep -E "sweep_I|mg_sweep|ms_per_step" | sed -e 's/.*ms_per_step": \([0-9.]*\).*/ms \1/' | awk '{printf "%s ", $0}')
  echo "$t :: $r"
done
