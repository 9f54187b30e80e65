timeout 900 python -m pytest tests/test_gpu_siddon.py -q -p no:cacheprovider 2>&1 | tail -15
timeout 300 python tools/time_ops.py --n 256 --angles 180
