mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
for v in "X=1" "FOCUS_B200_AGE_DIV=2" "FOCUS_B200_AGE_DIV=1" "FOCUS_B200_TCSPLIT=2" "FOCUS_B200_TCSPLIT=3"; do env $v timeout 90 python bench.py $Q > gpurun_out/bench_r02ay.log 2>&1; echo $v; grep '^{' gpurun_out/bench_r02ay.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); i=d['ingest']; print(d['value'], d['ms_per_step'], i['exact_rechecks'], i['resolve_profile']['fast_batches'])"; done
