mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
timeout 120 python bench.py $Q > gpurun_out/bench_r02aa.log 2>&1
grep '^{' gpurun_out/bench_r02aa.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
timeout 200 python tools/multi_probe.py --objects 1000000 --streams 1,2,4,8 --reps 6 > gpurun_out/multi_r02aa.log 2>&1
grep "^N=" gpurun_out/multi_r02aa.log
timeout 300 python -m pytest tests/test_gpu_shards.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_r02aa.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02aa.log; tail -2 gpurun_out/pytest_r02aa.log
