for v in default lists default lists; do
  if [ $v = default ]; then L=""; else L="build_variants/$v/libctk_b200.so"; fi
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 512 --angles 360 --reps 5
done
for v in default lists; do
  if [ $v = default ]; then L=""; else L="build_variants/$v/libctk_b200.so"; fi
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 256 --angles 180 --reps 7 --projector siddon
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 1024 --angles 200 --reps 3
done
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_siddon.py tests/test_gpu_golden.py tests/test_gpu_slab_band.py tests/test_gpu_slab.py tests/test_gpu_checked.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -3
