mkdir -p gpurun_out
timeout 600 python tools/c3_probe.py 300000 100000 5.0 > gpurun_out/c3_probe_r02f.log 2>&1
cat gpurun_out/c3_probe_r02f.log | cut -c1-900
