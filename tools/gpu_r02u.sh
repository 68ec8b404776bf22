mkdir -p gpurun_out
timeout 420 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r02u.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02u.log
tail -2 gpurun_out/pytest_r02u.log
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
timeout 150 python bench.py $Q > gpurun_out/bench_r02u.log 2>&1
FOCUS_B200_PREFETCH=0 timeout 150 python bench.py $Q > gpurun_out/bench_r02u_nopf.log 2>&1
timeout 150 python tools/trace_kernels.py > gpurun_out/trace_r02u_pdl.txt 2>&1
for f in gpurun_out/bench_r02u*.log; do echo $f; grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
sed -n '/^batch 150/,/^batch 151/p' gpurun_out/trace_r02u_pdl.txt
