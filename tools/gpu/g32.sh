timeout 600 python tools/time_bp.py --n 1024 --angles 400 --reps 3
CTK_BP_TILE=128 timeout 600 python tools/time_bp.py --n 1024 --angles 400 --reps 3
timeout 600 python bench.py --angles 45 --solver lsqr --no-cpu-baseline --steps 3 > gpurun_out/bench_rank45.json 2> gpurun_out/bench_rank45.err; tail -c 300 gpurun_out/bench_rank45.json
