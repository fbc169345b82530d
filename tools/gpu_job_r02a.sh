cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dist_native.py tests/test_gpu_dist.py -q -x > gpurun_out/dist_tests.log 2>&1; echo "dist tests exit $?"
tail -3 gpurun_out/dist_tests.log
timeout 600 python tools/panel_breakdown.py > gpurun_out/panel_breakdown.txt 2>&1; echo "panel exit $?"
timeout 900 python tools/dist_replay.py --out gpurun_out/dist_replay_cfg3.json > gpurun_out/dist_replay.log 2>&1; echo "replay exit $?"
tail -20 gpurun_out/dist_replay.log
rm -f gpurun_out/san/summary.txt
TOOLS="racecheck" CASES="lstsq qrglobal wide" bash tools/sanitize_all.sh
TOOLS="initcheck" CASES="lstsq gemm" bash tools/sanitize_all.sh
