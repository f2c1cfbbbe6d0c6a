# full ncu capture (source-level) of the first k_wave launch (M_II chain) with the library in tools/explibs/$1
mkdir -p gpurun_out
cp tools/explibs/$1/libspp.so paper_2108_13468_b200/lib/libspp.so
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
SPP_NO_GRAPH=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 0 -c 2 -o gpurun_out/prof_exp_$1 $CMD > gpurun_out/ncu_exp.log 2>&1
echo done
