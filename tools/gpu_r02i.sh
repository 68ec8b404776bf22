mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/box_r02i.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r02i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r02i.log
timeout 900 python bench.py > gpurun_out/bench_r02i.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r02i.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_r02i.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref_r02i.log
tail -3 gpurun_out/pytest_r02i.log; tail -c 3000 gpurun_out/bench_r02i.log
