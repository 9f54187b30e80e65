timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_r02b.log 2>&1; tail -3 gpurun_out/gputest_r02b.log
timeout 900 python bench.py > gpurun_out/bench_c3b.json 2> gpurun_out/bench_c3b.err; echo "c3 rc=$?"
timeout 600 python bench.py --config C1 --steps 300 > gpurun_out/bench_c1c.json 2> gpurun_out/bench_c1c.err; echo "c1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_atb_plane_f32 -c 1 -o gpurun_out/ncu_atb_r02b -f python tools/time_bp.py --reps 1 > gpurun_out/ncu_atb_b.log 2>&1; echo "ncu atb rc=$?"
