for v in default tab default tab; do
  if [ $v = default ]; then L=""; else L="build_variants/$v/libctk_b200.so"; fi
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 512 --angles 360 --reps 5
done
CTK_B200_LIB=build_variants/tab/libctk_b200.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "adjoint or atb" 2>&1 | tail -2
