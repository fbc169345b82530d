cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputest_r02x.log 2>&1; echo "gpu tests exit $?"
tail -4 gpurun_out/gputest_r02x.log
