timeout 300 python tools/time_bp.py --n 512 --angles 360 --reps 5
timeout 1800 python -m pytest tests/test_gpu_slab_band.py tests/test_gpu_slab.py tests/test_gpu_parity.py tests/test_gpu_checked.py tests/test_gpu_core.py -q -x -p no:cacheprovider 2>&1 | tail -3
