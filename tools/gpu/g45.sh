timeout 3300 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest_r02c.log 2>&1; tail -3 gpurun_out/gputest_r02c.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
