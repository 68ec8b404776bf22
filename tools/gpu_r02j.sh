mkdir -p gpurun_out
timeout 300 python tools/multi_probe.py --objects 1000000 --streams 1,2,4,8 --reps 2 > gpurun_out/multi_r02j_pdl.log 2>&1
FOCUS_B200_NOPDL=1 timeout 300 python tools/multi_probe.py --objects 1000000 --streams 1,2,4,8 --reps 2 > gpurun_out/multi_r02j_nopdl.log 2>&1
timeout 300 python tools/multi_probe.py --objects 1000000 --streams 8 --reps 1 --serial > gpurun_out/multi_r02j_serial.log 2>&1
timeout 300 python tools/multi_probe.py --objects 1000000 --streams 8 --reps 1 --trace 1 > gpurun_out/multi_r02j_trace.log 2>&1
tail -12 gpurun_out/multi_r02j_*.log
