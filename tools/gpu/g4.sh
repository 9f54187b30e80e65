nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1800 python -m pytest tests/test_gpu_core.py tests/test_gpu_checked.py -x -q -p no:cacheprovider 2>&1 | tail -5
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/gather_peak tools/gather_peak.cu && ./build/gather_peak 4096 > gpurun_out/gather_peak.json; cat gpurun_out/gather_peak.json
for c in C1 C2; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; tail -c 600 gpurun_out/bench_$c.json; done
