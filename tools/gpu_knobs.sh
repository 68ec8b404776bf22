mkdir -p gpurun_out
Q="--no-check --no-cpu --no-fc --multi-streams 1 --c3-objects 0 --queries 0 --e2e-steps 1 --steps 10 --warmup 3"
run() { env "$@" timeout 300 python bench.py $Q 2>/dev/null | grep '^{' | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$*', round(d['value']/1e6,2))" >> gpurun_out/knobs.log; }
run X=0
run FOCUS_B200_TFB_GY=128
run FOCUS_B200_TFB_GY=64
run FOCUS_B200_FOLD_GY=2
run FOCUS_B200_FOLD_GY=6
run X=0
run FOCUS_B200_TFB_GY=128
cat gpurun_out/knobs.log
