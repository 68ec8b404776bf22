mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seeds.py tests/test_gpu_scale_parity.py tests/test_gpu_reference_ports.py -x -q > gpurun_out/pytest_r02o.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02o.log
timeout 300 python tools/trace_kernels.py > gpurun_out/trace_r02o_pdl.txt 2>&1
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
for gy in 0 2 4 8; do FOCUS_B200_FOLD_GY=$gy timeout 300 python bench.py $Q > gpurun_out/bench_r02o_gy$gy.log 2>&1; done
FOCUS_B200_TFOLD_OLD=1 timeout 300 python bench.py $Q > gpurun_out/bench_r02o_old.log 2>&1
tail -3 gpurun_out/pytest_r02o.log
for f in gpurun_out/bench_r02o_*.log; do echo $f; grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('parity'))"; done
