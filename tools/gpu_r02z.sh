mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 170 python tools/multi_probe.py --objects 1000000 --streams 8 --reps 8 > gpurun_out/multi_r02z_$tag.log 2>&1; echo "== $tag rc=$?"; grep '^N=\|SLOW' gpurun_out/multi_r02z_$tag.log; }
run inline FOCUS_B200_FOLD_INLINE=1
run inline_nopdl FOCUS_B200_FOLD_INLINE=1 FOCUS_B200_NOPDL=1
run default X=1
