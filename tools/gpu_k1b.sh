mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fc_head.py tests/test_fc_oracle.py -x -q 2>&1 | tail -n 2 > gpurun_out/k1b_pytest12.log
for d in 0 0 16; do FOCUS_B200_FCDBG=$d timeout 200 python tools/ubench_fc2.py 2>&1 | grep -v -i warn | cut -c1-200 >> gpurun_out/k1b_ubench12.log; done
cat gpurun_out/k1b_pytest12.log gpurun_out/k1b_ubench12.log
