mkdir -p gpurun_out
timeout 200 python tools/multi_probe.py --objects 1000000 --streams 8 --reps 8 --partitions 8 > gpurun_out/multi_r02ab_p8.log 2>&1; echo "p8 rc=$?"
grep "^N=\|partitions\|SLOW\|Error\|error" gpurun_out/multi_r02ab_p8.log | head -20
timeout 200 python tools/multi_probe.py --objects 1000000 --streams 2 --reps 6 --partitions 2 > gpurun_out/multi_r02ab_p2.log 2>&1; echo "p2 rc=$?"
grep "^N=\|partitions\|SLOW\|Error\|error" gpurun_out/multi_r02ab_p2.log | head -20
timeout 200 python tools/multi_probe.py --objects 1000000 --streams 4 --reps 6 --partitions 4 > gpurun_out/multi_r02ab_p4.log 2>&1; echo "p4 rc=$?"
grep "^N=\|partitions\|SLOW\|Error\|error" gpurun_out/multi_r02ab_p4.log | head -20
