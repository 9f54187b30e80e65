timeout 300 python tools/time_bp.py --n 256 --angles 180 --projector siddon --reps 9
timeout 900 python -m pytest tests/test_gpu_siddon.py -q -x -p no:cacheprovider 2>&1 | tail -2
