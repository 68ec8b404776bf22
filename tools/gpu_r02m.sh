mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:k_tfold|k_rfast1|k_rfast3' --launch-skip 300 --launch-count 6 \
  -o gpurun_out/tfold_r02m -f python bench.py --steps 1 --warmup 0 --objects 300000 --no-cpu --no-check --e2e-steps 0 \
  --queries 0 --no-fc --multi-streams 0 --c3-objects 0 > gpurun_out/tfold_r02m.log 2>&1
echo done
