mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
for gy in 0 8 16; do FOCUS_B200_FOLD_GY=$gy timeout 120 python bench.py $Q > gpurun_out/bench_r02ag_$gy.log 2>&1; echo "gy=$gy"; grep '^{' gpurun_out/bench_r02ag_$gy.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
TAG=r02 timeout 1500 bash tools/gpu_profile_round.sh
ls -la gpurun_out/*r02.*
