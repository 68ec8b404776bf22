mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
for v in "X=1" "FOCUS_B200_FOLD_GY=4" "FOCUS_B200_FOLD_GY=8" "FOCUS_B200_FOLD_GY=2" "FOCUS_B200_NOPRIO=1"; do env $v timeout 90 python bench.py $Q > gpurun_out/bench_r02aq.log 2>&1; echo "$v"; grep '^{' gpurun_out/bench_r02aq.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
FOCUS_B200_FOLD_GY=4 timeout 60 python tools/trace_kernels.py > gpurun_out/trace_r02aq.txt 2>&1
grep -A11 "^batch" gpurun_out/trace_r02aq.txt | head -12
