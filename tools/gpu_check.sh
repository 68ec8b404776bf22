# Round check on one B200: GPU parity suite, smoke, default bench, reference arm.
mkdir -p gpurun_out
T=${TAG:-chk}
nvidia-smi > gpurun_out/smi_$T.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$T.log
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$T.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_$T.log
tail -n 3 gpurun_out/*_$T.log
