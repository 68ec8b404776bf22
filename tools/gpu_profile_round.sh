# Round profile set (1 GPU): launch list of one C2-prefix ingest, ncu --set full
# of the per-batch kernels at steady state, of the K1b head and of the
# feature-noise kernel.  TAG names the round.
mkdir -p gpurun_out
T=${TAG:-r02}
B="python bench.py --steps 1 --warmup 0 --objects 200000 --no-cpu --no-check --e2e-steps 0 --queries 0 --multi-streams 0 --c3-objects 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_$T.csv $B --no-fc > gpurun_out/launches_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_screen_tc|k_rowpass_lean|k_rfast|k_tfold_a4|k_tfold_b|k_fold|k_snap_pack|k_seal' --launch-skip 300 --launch-count 14 \
  -o gpurun_out/full_$T -f $B --no-fc > gpurun_out/full_$T.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_fc_tc|k_fc_merge|k_extract' --launch-count 3 \
  -o gpurun_out/fc_$T -f $B > gpurun_out/fc_$T.log 2>&1

timeout 600 python tools/trace_kernels.py 1000000 > gpurun_out/cupti_c2_$T.txt 2>&1
echo done
