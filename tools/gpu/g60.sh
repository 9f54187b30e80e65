# checked build: the pair suite; plus the pair tests on the normal build
timeout 1800 python -m pytest tests/test_gpu_checked.py -k pair -q 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_fwd_pair.py -q 2>&1 | tail -2
