mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool initcheck --print-limit 30 python tools/one_stream.py 60000 1004 > gpurun_out/san_initcheck_r02e.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 30 python tools/one_stream.py 60000 1004 > gpurun_out/san_memcheck_r02e.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 30 python tools/one_stream.py 30000 1004 7.5 100 4 > gpurun_out/san_memcheck4_r02e.log 2>&1
tail -5 gpurun_out/san_*_r02e.log
