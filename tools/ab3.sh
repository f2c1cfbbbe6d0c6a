# A/B of prebuilt libraries tools/ablibs/*.so: cfg4 per-class profile lines (given classes) and the cfg4 / cfg3 / cfg2 step times, interleaved
# usage: bash tools/ab3.sh "mg_prolong|mg_sweep"
CLS=${1:-"mg_prolong|mg_sweep|sweep_I"}
mkdir -p gpurun_out
for i in 1 2; do for v in $(ls tools/ablibs/*.so); do cp $v paper_2108_13468_b200/lib/libspp.so;
  r=$(timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-all 2>&1 | grep -E "$CLS|ms_per_step" | sed -e 's/.*ms_per_step": \([0-9.]*\).*/ms \1/' -e 's/launches= *[0-9]* //' -e 's/GB.*//' | awk '{printf "%s ", $0}')
  r3=$(timeout 200 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -o 'ms_per_step": [0-9.]*')
  r2=$(timeout 200 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -o 'ms_per_step": [0-9.]*')
  echo "$(basename $v) :: $r :: cfg3 $r3 :: cfg2 $r2"; done; done
