# Round profile set (1 GPU): launch list of one C2-prefix ingest + ncu --set full
# of the per-batch kernels at steady state and of the K1b head.  TAG names the round.
mkdir -p gpurun_out
T=${TAG:-r01}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 0 --objects 200000 --no-cpu \
  --e2e-steps 0 --queries 0 --no-fc > gpurun_out/launches_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_screen_tc|k_rowpass|k_resolve|k_fold|k_residuals' --launch-skip 150 --launch-count 10 \
  -o gpurun_out/full_$T -f python bench.py --steps 1 --warmup 0 --objects 200000 --no-cpu --e2e-steps 0 \
  --queries 0 --no-fc > gpurun_out/full_$T.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_fc_tc|k_fc_merge' --launch-count 2 \
  -o gpurun_out/fc_$T -f python bench.py --steps 1 --warmup 0 --objects 200000 --no-cpu --e2e-steps 0 \
  --queries 0 > gpurun_out/fc_$T.log 2>&1
echo done
