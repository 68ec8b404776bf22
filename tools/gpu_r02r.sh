mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
timeout 300 python bench.py $Q > gpurun_out/bench_r02r.log 2>&1
FOCUS_B200_NOPRIO=1 timeout 300 python bench.py $Q > gpurun_out/bench_r02r_noprio.log 2>&1
timeout 300 python tools/trace_kernels.py > gpurun_out/trace_r02r_pdl.txt 2>&1
timeout 300 python tools/multi_probe.py --objects 1000000 --streams 1,2,4,8 --reps 3 > gpurun_out/multi_r02r.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seeds.py tests/test_gpu_scale_parity.py -x -q > gpurun_out/pytest_r02r.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02r.log
tail -2 gpurun_out/pytest_r02r.log
for f in gpurun_out/bench_r02r*.log; do echo $f; grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
sed -n '/^batch 150/,/^batch 151/p' gpurun_out/trace_r02r_pdl.txt
grep "^N=" gpurun_out/multi_r02r.log
