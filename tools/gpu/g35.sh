for v in default b4m9 b2m18 b2m20 b8m4; do
  if [ $v = default ]; then L=""; else L="build_variants/$v/libctk_b200.so"; fi
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 512 --angles 360 --reps 5
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 256 --angles 180 --reps 7
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 1024 --angles 200 --reps 3
done
