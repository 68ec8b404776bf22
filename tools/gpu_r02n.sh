mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_noise.py -x -q > gpurun_out/pytest_noise_r02n.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_noise_r02n.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_r02n.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r02n.log
tail -5 gpurun_out/pytest_noise_r02n.log; tail -5 gpurun_out/pytest_r02n.log
