cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nullify.py tests/test_gpu_reuse.py -q -x > gpurun_out/svd_tests.log 2>&1; echo "tests exit $?"
tail -3 gpurun_out/svd_tests.log
timeout 300 python tools/panel_bench.py > gpurun_out/panel_bench_l.txt 2>&1; cat gpurun_out/panel_bench_l.txt
TOOLS="racecheck" CASES="lstsq" SAN_TIMEOUT=600 bash tools/sanitize_all.sh
grep SUMMARY gpurun_out/san/racecheck_lstsq.log
