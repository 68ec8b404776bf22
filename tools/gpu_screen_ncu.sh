mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_screen_tc -s 60 -c 1 -o gpurun_out/screen_r02f python tools/one_stream.py 400000 1004 > gpurun_out/screen_ncu.log 2>&1
tail -n 2 gpurun_out/screen_ncu.log
