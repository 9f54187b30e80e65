# final default bench line and the reference arm
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/g61_default.json 2> gpurun_out/g61_default.err; tail -c 400 gpurun_out/g61_default.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/g61_ref.json 2> gpurun_out/g61_ref.err; tail -c 400 gpurun_out/g61_ref.json
