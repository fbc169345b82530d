cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_fullpath.py tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -k "hqr or lstsq or cfg4" > gpurun_out/g16_tests.log 2>&1; echo "tests exit $?"
tail -5 gpurun_out/g16_tests.log
timeout 300 python tools/panel_breakdown.py 200000x256 150000x256 > gpurun_out/panel_breakdown_v.txt 2>&1; grep "==" gpurun_out/panel_breakdown_v.txt
