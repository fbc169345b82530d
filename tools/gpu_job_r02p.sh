cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dist_native.py -q -x > gpurun_out/dist_factor_tests.log 2>&1; echo "tests exit $?"
tail -25 gpurun_out/dist_factor_tests.log
