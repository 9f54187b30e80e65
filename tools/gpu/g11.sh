export CUDA_LAUNCH_BLOCKING=1
for v in wte wt7; do
  echo "== $v"
  CTK_B200_LIB=build_variants/$v/libctk_b200.so timeout 300 python tools/dbg_sid.py 256 180 joseph atb 2>&1 | tail -1
  CTK_B200_LIB=build_variants/$v/libctk_b200.so timeout 300 python tools/dbg_sid.py 512 360 joseph atb 2>&1 | tail -1
done
echo "== cur"; timeout 300 python tools/dbg_sid.py 512 360 joseph atb 2>&1 | tail -1
