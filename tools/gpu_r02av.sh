mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seeds.py tests/test_gpu_scale_parity.py -x -q > gpurun_out/pytest_r02av.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02av.log
tail -2 gpurun_out/pytest_r02av.log
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
for i in 1 2; do timeout 90 python bench.py $Q > gpurun_out/bench_r02av.log 2>&1; grep '^{' gpurun_out/bench_r02av.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
timeout 60 python tools/trace_kernels.py > gpurun_out/trace_r02av.txt 2>&1
grep -A11 "^batch" gpurun_out/trace_r02av.txt | head -12
