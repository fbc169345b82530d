cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_r02i.log 2>&1; echo "gpu tests exit $?"
tail -5 gpurun_out/gputest_r02i.log
timeout 300 python tools/panel_breakdown.py 50000x256 200000x256 > gpurun_out/panel_breakdown_i.txt 2>&1
grep "==" gpurun_out/panel_breakdown_i.txt
timeout 1500 python bench.py --config cfg4 --warmup 2 --steps 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_r02_cfg4.json 2> gpurun_out/bench_r02_cfg4.err; echo "cfg4 exit $?"
tail -c 400 gpurun_out/bench_r02_cfg4.json
timeout 1200 python bench.py --warmup 3 --steps 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_r02_cfg3_i.json 2> gpurun_out/bench_r02_cfg3_i.err; echo "cfg3 exit $?"
tail -c 300 gpurun_out/bench_r02_cfg3_i.json
