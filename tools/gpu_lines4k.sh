# TMA line chains at line length 4096 (cfg5): parity tests touching the lines, then cfg5/cfg4 benches
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "lines or region or cfg5 or cfg4 or precond or corner_solve" > gpurun_out/l4_tests.log 2>&1
timeout 600 python bench.py --config cfg5 --eps 1e-10 --no-cpu-baseline --no-e2e --profile-all > gpurun_out/l4_c5.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --profile-all > gpurun_out/l4_c4.log 2>&1
echo done
