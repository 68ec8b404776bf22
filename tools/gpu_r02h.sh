mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r02h.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r02h.log
timeout 600 python bench.py --steps 5 --warmup 3 --multi-streams 0 --no-check --no-cpu --queries 0 --no-fc > gpurun_out/bench_r02h.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r02h.log
FOCUS_B200_NOFAST=1 timeout 600 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 50 python tools/one_stream.py 8000 1004 > gpurun_out/san_racecheck_r02h.log 2>&1
timeout 600 compute-sanitizer --tool synccheck --print-limit 50 python tools/one_stream.py 8000 1004 > gpurun_out/san_synccheck_r02h.log 2>&1
tail -3 gpurun_out/pytest_r02h.log
