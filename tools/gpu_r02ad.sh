mkdir -p gpurun_out
Q="--steps 5 --warmup 3 --no-check --no-cpu --queries 0 --no-fc --multi-streams 0 --c3-objects 0 --e2e-steps 1"
for n in 0 8 16 24; do FOCUS_B200_CHAIN_SMS=$n timeout 120 python bench.py $Q > gpurun_out/bench_r02ad_$n.log 2>&1; echo "chain_sms=$n"; grep '^{' gpurun_out/bench_r02ad_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"; done
FOCUS_B200_CHAIN_SMS=16 timeout 120 python tools/trace_kernels.py > gpurun_out/trace_r02ad_pdl.txt 2>&1
sed -n '/^batch 150/,/^batch 151/p' gpurun_out/trace_r02ad_pdl.txt
