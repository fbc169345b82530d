cd $GRAFT_REPO_ROOT
timeout 1500 python tools/dist_replay.py --m 200000 --n 20000 --q 1 --k 16 --P 1 2 4 8 --out gpurun_out/dist_replay_cfg4.json > gpurun_out/dist_replay_cfg4.log 2>&1; echo "replay exit $?"
tail -4 gpurun_out/dist_replay_cfg4.log
