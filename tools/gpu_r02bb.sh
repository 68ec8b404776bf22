mkdir -p gpurun_out
Q="--steps 3 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 3"
for i in 1 2; do timeout 150 python bench.py $Q > gpurun_out/bench_r02bb.log 2>&1; grep '^{' gpurun_out/bench_r02bb.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])"; done
timeout 300 python -m pytest tests/test_gpu_reference_ports.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_r02bb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02bb.log; tail -2 gpurun_out/pytest_r02bb.log
