timeout 900 python tools/time_bp.py --n 1024 --angles 1600 --reps 2
CTK_BP_TILE=128 timeout 900 python tools/time_bp.py --n 1024 --angles 1600 --reps 2
CTK_BP_TILE=256 timeout 900 python tools/time_bp.py --n 512 --angles 720 --reps 3
timeout 900 python tools/time_bp.py --n 512 --angles 720 --reps 3
