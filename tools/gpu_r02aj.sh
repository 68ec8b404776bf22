mkdir -p gpurun_out
# multi-rank bench logic on one GPU: 2 ranks (gloo), both on cuda:0, smaller stream
FOCUS_B200_ONE_GPU=1 timeout 400 python bench.py --gpus 2 --backend gloo --steps 2 --warmup 1 --objects 200000 --no-cpu --queries 10 --c3-objects 0 --multi-streams 0 --e2e-steps 1 > gpurun_out/bench_r02aj_ws2.log 2>&1; echo "ws2 rc=$?"
grep '^{' gpurun_out/bench_r02aj_ws2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['value'], d['e2e']['value'], d['parity'] and d['parity']['mismatches'], d['query'])"
tail -5 gpurun_out/bench_r02aj_ws2.log | cut -c1-300
timeout 200 python bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_r02aj_ref2.log 2>&1; echo "ref2 rc=$?"; tail -2 gpurun_out/bench_r02aj_ref2.log | cut -c1-300
