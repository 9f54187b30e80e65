# parity + _core + sanitizer after the A^T b default change
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_core.py -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 300 python tools/time_bp.py --reps 7
for t in memcheck racecheck synccheck; do
  CTK_BP_TILE=128 timeout 900 compute-sanitizer --tool $t --print-limit 10 python tools/sanitize_cases.py joseph > gpurun_out/san_$t.log 2>&1; echo "$t rc=$?"; tail -3 gpurun_out/san_$t.log
done
CTK_BP_TILE=256 timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/sanitize_cases.py joseph > gpurun_out/san_rc256.log 2>&1; echo "rc256 rc=$?"; tail -3 gpurun_out/san_rc256.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python tools/sanitize_cases.py siddon > gpurun_out/san_sid.log 2>&1; echo "sid rc=$?"; tail -3 gpurun_out/san_sid.log
