mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_r02am.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02am.log
tail -3 gpurun_out/pytest_r02am.log
timeout 900 python bench.py > gpurun_out/bench_r02am.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r02am.log
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref_r02am.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_r02am.log
timeout 120 python tools/trace_kernels.py > gpurun_out/trace_r02am_pdl.txt 2>&1
grep '^{' gpurun_out/bench_r02am.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['parity']['mismatches'], d['multi_stream']['objects_per_s'], d['c5_query_sweep']['p50_ms'], d['c5_query_sweep']['parity'], d['k1b_fc_head']['frac'], d['feature_noise'], d['c3_shape']['objects_per_s'], d['roofline']['frac'])"
tail -c 400 gpurun_out/bench_ref_r02am.log
