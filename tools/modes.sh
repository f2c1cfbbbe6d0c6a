# A/B of environment modes on several configs: bash tools/modes.sh "cfg2 cfg3" "" "SPP_TUNE=coarse_max=32"
cfgs=$1; shift
for c in $cfgs; do for m in "$@"; do
 r=$(env $m python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config'].get('iters_per_solve'), d['gpu_launches'])")
 echo "$c [$m] $r"; done; done
