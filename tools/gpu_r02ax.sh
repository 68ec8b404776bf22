mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
for v in "X=1" "FOCUS_B200_TFB_GY=128" "FOCUS_B200_TFB_GY=64" "FOCUS_B200_TFB_GY=32"; do env $v timeout 90 python bench.py $Q > gpurun_out/bench_r02ax.log 2>&1; echo $v; grep '^{' gpurun_out/bench_r02ax.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
