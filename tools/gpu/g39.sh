for v in default kh2m3 kh2m4 default kh2m4; do
  if [ $v = default ]; then L=""; else L="build_variants/$v/libctk_b200.so"; fi
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 512 --angles 360 --reps 5
done
for v in default kh2m4; do
  if [ $v = default ]; then L=""; else L="build_variants/$v/libctk_b200.so"; fi
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 256 --angles 180 --reps 7
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 256 --angles 180 --reps 7 --projector siddon
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 64 --angles 100 --reps 9
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 512 --angles 720 --reps 3
done
CTK_B200_LIB=build_variants/kh2m4/libctk_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_siddon.py -q -x -p no:cacheprovider 2>&1 | tail -2
