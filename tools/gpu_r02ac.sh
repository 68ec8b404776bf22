mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --c3-objects 0 --e2e-steps 1"
timeout 300 python bench.py $Q > gpurun_out/bench_r02ac.log 2>&1
grep '^{' gpurun_out/bench_r02ac.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['multi_stream'])"
tail -3 gpurun_out/bench_r02ac.log | cut -c1-300
timeout 500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r02ac.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02ac.log
tail -3 gpurun_out/pytest_r02ac.log
