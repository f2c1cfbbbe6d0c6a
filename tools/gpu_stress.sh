# race check: the SPP_STRESS library (random delays at every k_wave hand-off) must reproduce the
# normal library's outputs bit for bit (tools/stress_check.py)
mkdir -p gpurun_out
timeout 600 python tools/stress_check.py save /tmp/stress_ref.npz > gpurun_out/stress.log 2>&1
cp tools/explibs/stress/libspp.so paper_2108_13468_b200/lib/libspp.so
timeout 1200 python tools/stress_check.py check /tmp/stress_ref.npz 3 >> gpurun_out/stress.log 2>&1
tail -5 gpurun_out/stress.log
