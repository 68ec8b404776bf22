mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r02ba.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02ba.log
tail -2 gpurun_out/pytest_r02ba.log
Q="--steps 3 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 3"
for i in 1 2; do timeout 150 python bench.py $Q > gpurun_out/bench_r02ba.log 2>&1; grep '^{' gpurun_out/bench_r02ba.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])"; done
