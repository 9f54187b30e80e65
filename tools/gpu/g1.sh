set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py "tests/test_gpu_fullsize.py::test_wide_offset_instantiation_matches" -x -q -p no:cacheprovider 2>&1 | tail -15
for v in default old p0 p1_12 p1_16 t0; do
  if [ $v = default ]; then timeout 300 python tools/time_bp.py --reps 7; else CTK_B200_LIB=build_variants/$v/libctk_b200.so timeout 300 python tools/time_bp.py --reps 7; fi
done
timeout 300 python tools/time_ops.py --n 256 --angles 180
