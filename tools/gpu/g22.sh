timeout 300 python tools/time_bp.py --n 512 --angles 360 --reps 7
CTK_B200_LIB=build_variants/c_bce3caa/libctk_b200.so timeout 300 python tools/time_bp.py --n 512 --angles 360 --reps 7
timeout 300 python tools/time_bp.py --n 64 --angles 100 --reps 9
CTK_BP_TILE=128 timeout 300 python tools/time_bp.py --n 64 --angles 100 --reps 9
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_fullsize.py tests/test_gpu_slab_band.py -q -x -p no:cacheprovider 2>&1 | tail -3
