# ncu --set full of the two-volume march (chunk 0) at C3
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ax2_zfast -c 1 -f -o gpurun_out/ax2_512 python tools/solve_once.py --n 512 --angles 360 --iters 2 --reps 1 > gpurun_out/g51.log 2>&1; tail -3 gpurun_out/g51.log
