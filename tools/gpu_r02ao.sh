mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
timeout 120 python bench.py $Q > gpurun_out/bench_r02ao.log 2>&1
FOCUS_B200_RP_LEAN=0 timeout 120 python bench.py $Q > gpurun_out/bench_r02ao_old.log 2>&1
for f in gpurun_out/bench_r02ao*.log; do echo $f; grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['per_kernel']['screen_summary']['ms_per_step'])"; done
timeout 120 python tools/trace_kernels.py > gpurun_out/trace_r02ao.txt 2>&1
grep -A11 "^batch" gpurun_out/trace_r02ao.txt | head -12
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seeds.py tests/test_gpu_scale_parity.py -x -q > gpurun_out/pytest_r02ao.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02ao.log
tail -2 gpurun_out/pytest_r02ao.log
