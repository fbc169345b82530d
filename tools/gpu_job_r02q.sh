cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputest_r02q.log 2>&1; echo "gpu tests exit $?"
tail -4 gpurun_out/gputest_r02q.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
