mkdir -p gpurun_out
nproc > gpurun_out/box_r02b.txt; free -g >> gpurun_out/box_r02b.txt
timeout 300 python tools/multi_probe.py --objects 1000000 --streams 1,2,4,8 > gpurun_out/multi_r02b_pdl.log 2>&1
FOCUS_B200_NOPDL=1 timeout 300 python tools/multi_probe.py --objects 1000000 --streams 1,2,4,8 > gpurun_out/multi_r02b_nopdl.log 2>&1
timeout 300 python tools/multi_probe.py --objects 1000000 --streams 8 --serial > gpurun_out/multi_r02b_serial.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_scale_parity.py -x -q -s > gpurun_out/scale_parity_r02b.log 2>&1
tail -3 gpurun_out/*_r02b*.log
