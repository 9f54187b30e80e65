# A/B timing of matched A^T b variants (build_variants/*), plus ncu of two of them
for v in A B C D E; do
  CTK_B200_LIB=build_variants/$v/libctk_b200.so timeout 300 python tools/time_bp.py --reps 7
done
for v in A C; do
  CTK_B200_LIB=build_variants/$v/libctk_b200.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_atb_plane_f32 -c 1 -o gpurun_out/ncu_atb_$v -f python tools/time_bp.py --reps 1 > gpurun_out/ncu_atb_$v.log 2>&1
done
