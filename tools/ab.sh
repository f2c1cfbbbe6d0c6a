# A/B of prebuilt libraries in tools/ablibs/*.so on the cfg4 bench (same box, interleaved)
for i in 1 2; do for v in $(ls tools/ablibs/*.so); do cp $v paper_2108_13468_b200/lib/libspp.so;
  r=$(timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-all 2>&1 | grep -E "sweep_I|mg_sweep|ms_per_step" | sed -e 's/.*ms_per_step": \([0-9.]*\).*/ms \1/' | awk '{printf "%s ", $0}')
  echo "$(basename $v) :: $r"; done; done
