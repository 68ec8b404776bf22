mkdir -p gpurun_out
for d in 0 16 32 48 4; do FOCUS_B200_FCDBG=$d timeout 200 python tools/ubench_fc2.py 2>&1 | grep -v -i warn | cut -c1-200 >> gpurun_out/k1b_ubench10.log; done
cat gpurun_out/k1b_ubench10.log
