mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" FOCUS_B200_STALL=300 timeout 150 python tools/multi_probe.py --objects 1000000 --streams 1,8 --reps 4 > gpurun_out/multi_r02v_$tag.log 2>&1; echo "== $tag rc=$?"; grep '^N=' gpurun_out/multi_r02v_$tag.log; grep -c STALL gpurun_out/multi_r02v_$tag.log; }
run default X=1
run gy4 FOCUS_B200_FOLD_GY=4
run gy2 FOCUS_B200_FOLD_GY=2
run gy4nopdl FOCUS_B200_FOLD_GY=4 FOCUS_B200_NOPDL=1
