mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
for bm in 4096 8192 16384; do FOCUS_B200_BMAX=$bm timeout 150 python bench.py $Q > gpurun_out/bench_r02ai_$bm.log 2>&1; echo "bmax=$bm"; grep '^{' gpurun_out/bench_r02ai_$bm.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); i=d['ingest']; print(d['value'], d['ms_per_step'], i['fast_decisions'], i['resolve_profile']['fast_batches'], i['exact_rechecks'])"; tail -2 gpurun_out/bench_r02ai_$bm.log | cut -c1-200; done
FOCUS_B200_BMAX=8192 timeout 600 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py tests/test_gpu_seeds.py -x -q > gpurun_out/pytest_r02ai.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02ai.log
tail -3 gpurun_out/pytest_r02ai.log
