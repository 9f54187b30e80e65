nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_r02.log 2>&1; tail -3 gpurun_out/gputest_r02.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --config C1 --steps 100 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "c1 rc=$?"
timeout 900 python bench.py --config C2 --steps 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout 1500 python bench.py --config C4 --steps 2 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 3 --iters 5 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_atb_plane_f32 -c 1 -o gpurun_out/ncu_atb_r02 -f python tools/time_bp.py --reps 1 > gpurun_out/ncu_atb.log 2>&1; echo "ncu atb rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ax_zfast_f32 -c 1 -o gpurun_out/ncu_ax_r02 -f python tools/time_bp.py --reps 1 > gpurun_out/ncu_ax.log 2>&1; echo "ncu ax rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_atb_plane_f32 -c 1 -o gpurun_out/ncu_sid_atb_r02 -f python tools/time_bp.py --n 256 --angles 180 --projector siddon --reps 1 > gpurun_out/ncu_sid.log 2>&1; echo "ncu sid rc=$?"
