for v in default b4 b4m9 b4m10 b4m12 default b4m9 b4m10; do
  if [ $v = default ]; then L=""; else L="build_variants/$v/libctk_b200.so"; fi
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 512 --angles 360 --reps 5
done
