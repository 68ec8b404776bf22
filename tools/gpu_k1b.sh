mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fc_head.py tests/test_fc_oracle.py -x -q 2>&1 | tail -n 2 > gpurun_out/k1b_pytest15.log
for v in "1 4" "1 2" "0 4"; do set -- $v; FOCUS_B200_FC_W64=$1 FOCUS_B200_FC_LD=$2 timeout 200 python tools/ubench_fc2.py 2>&1 | grep -v -i warn | cut -c1-300 >> gpurun_out/k1b_ubench15.log; done
cat gpurun_out/k1b_pytest15.log gpurun_out/k1b_ubench15.log
