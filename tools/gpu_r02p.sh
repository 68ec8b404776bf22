mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
timeout 300 python bench.py $Q > gpurun_out/bench_r02p.log 2>&1
FOCUS_B200_FOLD_GY=4 timeout 300 python bench.py $Q > gpurun_out/bench_r02p_gy4.log 2>&1
timeout 300 python tools/trace_kernels.py > gpurun_out/trace_r02p_pdl.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_tfold2' --launch-skip 150 --launch-count 2 \
  -o gpurun_out/tfold2_r02p -f python tools/trace_kernels.py 300000 > gpurun_out/tfold2_r02p.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_seeds.py tests/test_gpu_scale_parity.py -x -q > gpurun_out/pytest_r02p.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02p.log
tail -2 gpurun_out/pytest_r02p.log
for f in gpurun_out/bench_r02p*.log; do echo $f; grep '^{' $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
