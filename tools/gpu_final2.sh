# Round-2 measurement: parity tests, smoke, the default bench line (cfg4, with e2e and the CPU
# baseline), the reference arm (the oracle), the other BASELINE configs, the ncu launch list, the
# DRAM bytes of every k_wave launch, and ncu --set full captures of the top kernels.
O=gpurun_out/final2
mkdir -p $O/configs
nvidia-smi > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --profile-all > $O/bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1; echo "ref rc=$?"
for e in 1e-10 1e-8 1e-6; do timeout 900 python bench.py --config cfg5 --eps $e --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --profile-all > $O/configs/cfg5_$e.log 2>&1; done
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-all > $O/configs/cfg3.log 2>&1
timeout 600 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --profile-all > $O/configs/cfg2.log 2>&1
timeout 600 python bench.py --config cfg1-batch > $O/configs/cfg1_batch.log 2>&1
timeout 900 python bench.py --config cfg5-sweep --steps 1 --warmup 1 > $O/configs/cfg5_sweep.log 2>&1
timeout 600 python tools/paper_times.py > $O/paper_table7_times.txt 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
# ncu runs use the host-driven corner loop (SPP_NO_GRAPH=1): the same kernels, one launch each
SPP_NO_GRAPH=1 $CMD > $O/plain.log 2>&1 && \
SPP_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file $O/launches.csv $CMD > $O/ncu_list.log 2>&1
SPP_NO_GRAPH=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_wave -c 1000 --csv --log-file $O/wave_dram.csv $CMD > $O/ncu_dram.log 2>&1
SPP_NO_GRAPH=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 0 -c 3 -o $O/prof_wave $CMD > $O/ncu_full.log 2>&1
SPP_NO_GRAPH=1 timeout 1200 ncu --set full --clock-control none -k regex:"k_lines_tma|k_cycle_update|k_resid_restrict|k_gs_prep|k_spmv|k_mgs|k_corner_rhs|k_coarse_vcycle" -c 10 -o $O/prof_other $CMD > $O/ncu_other.log 2>&1
ls -la $O
echo done
