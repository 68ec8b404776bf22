mkdir -p gpurun_out
FOCUS_B200_NOPDL=1 timeout 300 python tools/trace_kernels.py > gpurun_out/trace_r02l_nopdl.txt 2>&1
timeout 300 python tools/trace_kernels.py > gpurun_out/trace_r02l_pdl.txt 2>&1
TAG=r02l bash tools/gpu_profile_round.sh
ls -la gpurun_out
