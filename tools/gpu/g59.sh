# final: full GPU suite + smoke
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/g59_tests.log 2>&1; tail -3 gpurun_out/g59_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
