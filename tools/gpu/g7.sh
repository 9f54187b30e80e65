timeout 300 python tools/time_ops.py --n 256 --angles 180 2>&1 | tail -12
