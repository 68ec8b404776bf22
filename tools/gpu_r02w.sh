mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_screen_tc.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_r02w.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02w.log
tail -3 gpurun_out/pytest_r02w.log
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
timeout 120 python bench.py $Q > gpurun_out/bench_r02w.log 2>&1
FOCUS_B200_TC2=0 timeout 120 python bench.py $Q > gpurun_out/bench_r02w_tc1.log 2>&1
timeout 120 python tools/trace_kernels.py > gpurun_out/trace_r02w_pdl.txt 2>&1
for f in gpurun_out/bench_r02w*.log; do echo $f; grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; tail -2 $f; done
sed -n '/^batch 150/,/^batch 151/p' gpurun_out/trace_r02w_pdl.txt
timeout 150 python tools/multi_probe.py --objects 1000000 --streams 8 --reps 5 > gpurun_out/multi_r02w.log 2>&1
grep "^N=\|SLOW" gpurun_out/multi_r02w.log
