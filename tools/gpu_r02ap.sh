mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
timeout 90 python bench.py $Q > gpurun_out/bench_r02ap.log 2>&1; echo "bench rc=$?"
grep '^{' gpurun_out/bench_r02ap.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
timeout 60 python tools/trace_kernels.py > gpurun_out/trace_r02ap.txt 2>&1; echo "trace rc=$?"
grep -A11 "^batch" gpurun_out/trace_r02ap.txt | head -12
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seeds.py tests/test_gpu_scale_parity.py tests/test_gpu_partitions.py -x -q > gpurun_out/pytest_r02ap.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02ap.log
tail -2 gpurun_out/pytest_r02ap.log
timeout 120 python tools/multi_probe.py --objects 1000000 --streams 2 --reps 3 > gpurun_out/multi_r02ap.log 2>&1; echo "multi rc=$?"; grep "^N=" gpurun_out/multi_r02ap.log
