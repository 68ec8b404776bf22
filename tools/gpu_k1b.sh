mkdir -p gpurun_out
for r in 1 0; do FOCUS_B200_FC_MERGE_REG=$r timeout 200 python tools/ubench_fc2.py 2>&1 | grep -v -i warn >> gpurun_out/k1b_ubench4.log; done
FOCUS_B200_FCDBG=4 timeout 200 python tools/ubench_fc2.py 2>&1 | grep -v -i warn | cut -c1-300 >> gpurun_out/k1b_ubench4.log
cat gpurun_out/k1b_ubench4.log
