mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r02f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r02f.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r02f.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r02f.log
FOCUS_B200_CHECK=1 timeout 600 python tools/multi_probe.py --objects 1000000 --streams 8 --reps 3 --counters > gpurun_out/multi_r02f_check.log 2>&1
tail -3 gpurun_out/pytest_r02f.log
