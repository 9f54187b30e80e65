# two-volume march: tests, then occupancy / unroll variants via time_pair
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fwd_pair.py -x -q 2>&1 | tail -3
for v in default p6 p7 p9 u2 u2m6; do
  if [ $v = default ]; then L=paper_2211_14212_b200/lib/libctk_b200.so; else L=build_variants/$v/libctk_b200.so; fi
  for cfg in "512 360" "256 180" "512 45"; do
    set -- $cfg
    echo "$v $(CTK_B200_LIB=$L timeout 300 python tools/time_pair.py --n $1 --angles $2 2>&1 | tail -1)"
  done
done
