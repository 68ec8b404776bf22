mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r02t.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02t.log
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
timeout 300 python bench.py $Q > gpurun_out/bench_r02t.log 2>&1
timeout 300 python tools/trace_kernels.py > gpurun_out/trace_r02t_pdl.txt 2>&1
FOCUS_B200_STALL=200 timeout 400 python tools/multi_probe.py --objects 1000000 --streams 1,2,4,8 --reps 3 --trace-stall 3 > gpurun_out/multi_r02t.log 2>&1
tail -2 gpurun_out/pytest_r02t.log
for f in gpurun_out/bench_r02t*.log; do echo $f; grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
sed -n '/^batch 150/,/^batch 151/p' gpurun_out/trace_r02t_pdl.txt
grep -v Warn gpurun_out/multi_r02t.log | grep -v "^ *_warn" | tail -30
