# ncu --set full of selected kernels at steady state (1 GPU): KERNELS regex, TAG
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on ${NCU_EXTRA:-} \
  -k "regex:${KERNELS:-k_fold|k_resolve}" --launch-skip ${SKIP:-100} --launch-count ${COUNT:-4} \
  -o gpurun_out/full_${TAG:-k} -f python bench.py --steps 1 --warmup 0 --objects ${NOBJ:-200000} --no-cpu --e2e-steps 0 \
  > gpurun_out/ncu_${TAG:-k}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_${TAG:-k}.log
