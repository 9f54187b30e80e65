export CUDA_LAUNCH_BLOCKING=1
for n in 64 128 256; do timeout 300 python tools/dbg_sid.py $n 180 joseph atb 2>&1 | tail -1; done
timeout 300 python tools/dbg_sid.py 256 180 joseph ax atb 2>&1 | tail -1
timeout 300 python tools/dbg_sid.py 256 64 joseph atb 2>&1 | tail -1
timeout 300 python tools/dbg_sid.py 512 360 joseph atb 2>&1 | tail -1
CTK_BP_TILE=256 timeout 300 python tools/dbg_sid.py 256 180 joseph atb 2>&1 | tail -1
