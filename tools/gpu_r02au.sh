mkdir -p gpurun_out
timeout 500 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_seeds.py -x -q > gpurun_out/pytest_r02au.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02au.log
tail -2 gpurun_out/pytest_r02au.log
Q="--steps 3 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --e2e-steps 1"
timeout 300 python bench.py $Q > gpurun_out/bench_r02au.log 2>&1
FOCUS_B200_TCLOAD=cp timeout 300 python bench.py $Q > gpurun_out/bench_r02au_cp.log 2>&1
for f in gpurun_out/bench_r02au*.log; do echo $f; grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['c3_shape']['objects_per_s'])"; done
timeout 200 python tools/trace_kernels.py 300000 5.0 100000 > gpurun_out/trace_c3_r02au.txt 2>&1
grep -A12 "^batch" gpurun_out/trace_c3_r02au.txt | head -13
