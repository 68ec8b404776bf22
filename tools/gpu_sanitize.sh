# compute-sanitizer over the hot path (racecheck / synccheck on the
# race-prone kernels k_resolve, k_fold / k_tfold, K3 atomics; memcheck, initcheck)
mkdir -p gpurun_out
S="compute-sanitizer --print-limit 20 --error-exitcode 9"
run() { name=$1; shift; timeout 900 $S "$@" > gpurun_out/san_$name.log 2>&1; echo "rc=$?" >> gpurun_out/san_$name.log; }
run racecheck_c2   --tool racecheck --racecheck-report all python tools/one_stream.py 12000 1004
run synccheck_c2   --tool synccheck python tools/one_stream.py 12000 1004
run memcheck_c2    --tool memcheck  python tools/one_stream.py 40000 1004
run racecheck_evict --tool racecheck --racecheck-report all python tools/one_stream.py 6000 1005 5.0 500
run memcheck_evict --tool memcheck python tools/one_stream.py 20000 1005 5.0 500
run initcheck_c2   --tool initcheck python tools/one_stream.py 20000 1004
N=2048 run racecheck_fc --tool racecheck --racecheck-report all python tools/ubench_fc2.py
N=8192 run memcheck_fc --tool memcheck python tools/ubench_fc2.py
for f in gpurun_out/san_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=" $f | tail -n 3; done
