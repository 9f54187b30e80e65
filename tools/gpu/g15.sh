timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py tests/test_gpu_siddon.py tests/test_gpu_operators.py -q -x -p no:cacheprovider 2>&1 | tail -3
