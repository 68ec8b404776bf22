mkdir -p gpurun_out
Q="--no-check --no-cpu --no-fc --multi-streams 1 --c3-objects 0 --queries 0 --e2e-steps 1 --steps 10 --warmup 3"
timeout 600 python -m pytest tests/test_gpu_screen_tc.py tests/test_gpu_scale_parity.py tests/test_gpu_parity.py -x -q 2>&1 | tail -n 2 > gpurun_out/scr_pytest.log
for t in 1 0 1 0; do FOCUS_B200_TC2=$t timeout 300 python bench.py $Q 2>/dev/null | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('TC2=$t', round(d['value']/1e6,2), d['roofline']['avg_launch_us'], d['roofline']['phase_ms_per_step'])" >> gpurun_out/scr_bench.log; done
cat gpurun_out/scr_pytest.log gpurun_out/scr_bench.log
