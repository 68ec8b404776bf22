mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r02g.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r02g.log
timeout 600 python tools/multi_probe.py --objects 1000000 --streams 2,8 --reps 3 --verify --counters > gpurun_out/multi_r02g_verify.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --multi-streams 0 > gpurun_out/bench_r02g.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r02g.log
timeout 900 compute-sanitizer --tool initcheck --print-limit 200 python tools/one_stream.py 20000 1004 > gpurun_out/san_initcheck_r02g.log 2>&1
tail -3 gpurun_out/pytest_r02g.log
