timeout 1500 python -m pytest tests/test_gpu_slab_band.py tests/test_gpu_slab.py -q -x -p no:cacheprovider 2>&1 | tail -30
