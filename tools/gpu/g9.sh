CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/time_ops.py --n 256 --angles 180 2>&1 | grep -v "^  \|^\[W" | tail -8
CTK_B200_LIB=paper_2211_14212_b200/lib/checked/libctk_b200.so CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/time_ops.py --n 256 --angles 180 2>&1 | grep -v "^  \|^\[W" | tail -8
