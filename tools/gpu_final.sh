# Round measurement: parity tests, smoke, default bench line, launch list, DRAM traffic of every
# MG-sweep launch of one solve, and one full ncu capture of the first k_wave launches.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --profile-all > gpurun_out/bench.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
# ncu runs use the host-driven corner loop (SPP_NO_GRAPH=1): the same kernels, one launch each
SPP_NO_GRAPH=1 $CMD > gpurun_out/plain.log 2>&1 && \
SPP_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu.log 2>&1
SPP_NO_GRAPH=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_wave -c 1000 --csv --log-file gpurun_out/wave_dram.csv $CMD > gpurun_out/ncu_dram.log 2>&1
SPP_NO_GRAPH=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_wave -s 0 -c 3 -o gpurun_out/prof_final $CMD > gpurun_out/ncu_full.log 2>&1
echo done
