cd $GRAFT_REPO_ROOT
timeout 600 python tools/panel_breakdown.py 50000x256 200000x256 20000x256 > gpurun_out/panel_breakdown_b.txt 2>&1; echo "panel exit $?"
grep "==" gpurun_out/panel_breakdown_b.txt
timeout 900 python -m pytest tests/test_gpu_dist_native.py tests/test_gpu_parity.py tests/test_gpu_fullpath.py -q -x > gpurun_out/tests_b.log 2>&1; echo "tests exit $?"
tail -3 gpurun_out/tests_b.log
