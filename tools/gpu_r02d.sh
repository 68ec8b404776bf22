mkdir -p gpurun_out
timeout 300 python tools/multi_probe.py --objects 1000000 --streams 1,8 --reps 3 --counters > gpurun_out/multi_r02d_cnt.log 2>&1
FOCUS_B200_NOPDL=1 timeout 300 python tools/multi_probe.py --objects 1000000 --streams 8 --reps 2 --trace 1 > gpurun_out/multi_r02d_nopdl_trace.log 2>&1
timeout 600 python -m pytest tests/test_gpu_shards.py -x -q > gpurun_out/pytest_shards_r02d.log 2>&1
tail -3 gpurun_out/pytest_shards_r02d.log
