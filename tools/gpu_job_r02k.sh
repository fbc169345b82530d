cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_dist_procs.py tests/test_gpu_dist_ooc.py -q -x > gpurun_out/dist_procs_tests.log 2>&1; echo "tests exit $?"
tail -30 gpurun_out/dist_procs_tests.log
timeout 900 python bench.py --config cfg2 --streamed 0 --force-dist --warmup 1 --steps 1 > gpurun_out/bench_r02_streamed_dist_cfg2.json 2> gpurun_out/bench_r02_streamed_dist_cfg2.err; echo "streamed dist bench exit $?"
tail -c 800 gpurun_out/bench_r02_streamed_dist_cfg2.json
tail -5 gpurun_out/bench_r02_streamed_dist_cfg2.err
