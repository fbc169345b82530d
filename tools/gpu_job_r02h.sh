cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dist_ooc.py -q -x > gpurun_out/dist_ooc_tests.log 2>&1; echo "dist ooc tests exit $?"
tail -25 gpurun_out/dist_ooc_tests.log
timeout 900 python -m pytest tests/test_gpu_fullpath.py tests/test_gpu_parity.py -q -x -k "hqr or lstsq" > gpurun_out/hqr_tests.log 2>&1; echo "hqr tests exit $?"
tail -3 gpurun_out/hqr_tests.log
timeout 300 python tools/panel_breakdown.py 50000x256 20000x256 200000x256 > gpurun_out/panel_breakdown_h.txt 2>&1
grep "==" gpurun_out/panel_breakdown_h.txt
UTV_TRACE=1 python -c 'from paper_2408_05238_b200 import build as b; b.build(force=True)' > /dev/null 2>&1
for m in 50000 20000 200000; do python tools/qr_phase_trace.py $m; done
