mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r02c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r02c.log
timeout 400 python tools/multi_probe.py --objects 1000000 --streams 8 --reps 3 --trace 2 > gpurun_out/multi_r02c_trace.log 2>&1
tail -3 gpurun_out/pytest_r02c.log
