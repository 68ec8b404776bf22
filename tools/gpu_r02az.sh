mkdir -p gpurun_out
Q="--steps 3 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 3"
for v in "FOCUS_B200_H2D_MB=1024" "X=1" "FOCUS_B200_H2D_MB=128" "FOCUS_B200_H2D_MB=64"; do env $v timeout 150 python bench.py $Q > gpurun_out/bench_r02az.log 2>&1; echo $v; grep '^{' gpurun_out/bench_r02az.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'])"; done
