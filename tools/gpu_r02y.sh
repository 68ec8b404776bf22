mkdir -p gpurun_out
timeout 500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r02y.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02y.log
tail -3 gpurun_out/pytest_r02y.log
timeout 900 python bench.py > gpurun_out/bench_r02y.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r02y.log
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref_r02y.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_r02y.log
grep '^{' gpurun_out/bench_r02y.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d.get('parity',{}).get('mismatches'), d.get('multi_stream'), d.get('c5_query_sweep',{}).get('parity'))"
tail -c 600 gpurun_out/bench_ref_r02y.log
