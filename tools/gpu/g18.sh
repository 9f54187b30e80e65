for v in default c_bce3caa c_eca2f15; do
  if [ $v = default ]; then L=""; else L="build_variants/$v/libctk_b200.so"; fi
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 512 --angles 360 --reps 5
done
timeout 600 python -m pytest tests/test_gpu_slab_band.py -q -x -p no:cacheprovider 2>&1 | tail -2
