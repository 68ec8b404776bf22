mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 240 python tools/multi_probe.py --objects 1000000 --streams 8 --reps 4 > gpurun_out/multi_r02k_$tag.log 2>&1; echo "== $tag rc=$?"; grep '^N=' gpurun_out/multi_r02k_$tag.log; }
run split1 FOCUS_B200_TCSPLIT=1
run conn32 CUDA_DEVICE_MAX_CONNECTIONS=32
run conn32split1 CUDA_DEVICE_MAX_CONNECTIONS=32 FOCUS_B200_TCSPLIT=1
run nopdl_split1 FOCUS_B200_NOPDL=1 FOCUS_B200_TCSPLIT=1
run default X=1
