# GPU parity tests + one bench line (1 GPU); outputs under gpurun_out/
mkdir -p gpurun_out
T=${TAG:-q}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 600 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench_$T.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$T.log
tail -3 gpurun_out/pytest_$T.log
grep '^{' gpurun_out/bench_$T.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['phase_ms_per_step'], d['e2e']['value'] if d.get('e2e') else None)"
if [ -n "$LAUNCHES" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 0 --objects 200000 --no-cpu --e2e-steps 0 > /dev/null 2>&1
python tools/ncu_launch_summary.py gpurun_out/launches_$T.csv | head -14
fi
