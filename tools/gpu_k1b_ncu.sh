mkdir -p gpurun_out
N=65536 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fc_merge -c 1 -o gpurun_out/k1b_merge python tools/ubench_fc2.py > gpurun_out/k1b_ncu2.log 2>&1
tail -n 3 gpurun_out/k1b_ncu2.log
