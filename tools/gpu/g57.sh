# slice chunks for the two-volume march (CTK_FWD_CHUNKS applies to both marches)
for cfg in "512 360" "512 45" "256 180" "1024 200"; do
  set -- $cfg
  for c in 1 2 4 8; do
    echo "chunks=$c $(CTK_FWD_CHUNKS=$c timeout 300 python tools/time_pair.py --n $1 --angles $2 --reps 3 2>&1 | tail -1)"
  done
done
