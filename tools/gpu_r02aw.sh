mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
for v in "X=1" "FOCUS_B200_TF4=0"; do env $v timeout 90 python bench.py $Q > gpurun_out/bench_r02aw.log 2>&1; echo $v; grep '^{' gpurun_out/bench_r02aw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
timeout 60 python tools/trace_kernels.py > gpurun_out/trace_r02aw.txt 2>&1
grep -A11 "^batch" gpurun_out/trace_r02aw.txt | head -12
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seeds.py tests/test_gpu_scale_parity.py -x -q > gpurun_out/pytest_r02aw.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02aw.log
tail -2 gpurun_out/pytest_r02aw.log
