for v in default bc8; do
  if [ $v = default ]; then L=""; else L="build_variants/$v/libctk_b200.so"; fi
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 256 --angles 180 --reps 7 --projector siddon
  CTK_B200_LIB=$L timeout 300 python tools/time_bp.py --n 64 --angles 100 --reps 9
done
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_siddon.py tests/test_gpu_slab.py tests/test_gpu_slab_band.py tests/test_gpu_fullsize.py tests/test_gpu_checked.py -q -x -p no:cacheprovider 2>&1 | tail -2
