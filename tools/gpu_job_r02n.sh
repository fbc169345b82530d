cd $GRAFT_REPO_ROOT
timeout 900 python tools/dist_replay.py --out gpurun_out/dist_replay_cfg3_r02n.json > gpurun_out/dist_replay_n.log 2>&1; echo "replay exit $?"
timeout 600 python tools/dist_replay.py --P 2 4 8 --chunks 1 --out gpurun_out/dist_replay_cfg3_chunks1.json > gpurun_out/dist_replay_c1.log 2>&1; echo "replay c1 exit $?"
tail -3 gpurun_out/dist_replay_n.log gpurun_out/dist_replay_c1.log
