mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fc_head.py tests/test_fc_oracle.py -x -q 2>&1 | tail -n 2 > gpurun_out/k1b_pytest11.log
for l in 4 2 4 2; do FOCUS_B200_FC_LD=$l timeout 200 python tools/ubench_fc2.py 2>&1 | grep -v -i warn | cut -c1-200 >> gpurun_out/k1b_ubench11.log; done
cat gpurun_out/k1b_pytest11.log gpurun_out/k1b_ubench11.log
