# one ncu --set full capture of the per-batch ingest kernels at steady state (1 GPU)
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_resolve|k_fold|k_screen|k_row_summary|k_residuals' --launch-skip 200 --launch-count 10 \
  -o gpurun_out/full_${TAG:-r1} -f python bench.py --steps 1 --warmup 0 --objects 200000 --no-cpu --e2e-steps 0 \
  > gpurun_out/ncu_full_${TAG:-r1}.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_${TAG:-r1}.log
