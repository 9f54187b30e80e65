for v in default s1 s2; do
  if [ $v = default ]; then L=""; else L="build_variants/$v/libctk_b200.so"; fi
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 256 --angles 180 --projector siddon --reps 9
done
timeout 300 python tools/time_bp.py --n 512 --angles 360 --projector siddon --reps 5
