for v in default dense default dense; do
  if [ $v = default ]; then L=""; else L="build_variants/$v/libctk_b200.so"; fi
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 512 --angles 360 --reps 5
done
for v in default dense; do
  if [ $v = default ]; then L=""; else L="build_variants/$v/libctk_b200.so"; fi
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 256 --angles 180 --reps 7
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 1024 --angles 1600 --reps 1
done
CTK_B200_LIB=build_variants/dense/libctk_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -2
