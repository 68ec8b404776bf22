mkdir -p gpurun_out
FOCUS_B200_STALL=200 timeout 600 python tools/multi_probe.py --objects 1000000 --streams 8 --reps 6 --trace-stall 6 > gpurun_out/multi_r02s.log 2>&1
grep -v Warn gpurun_out/multi_r02s.log | tail -40
