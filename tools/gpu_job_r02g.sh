cd $GRAFT_REPO_ROOT
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 12000 --log-file gpurun_out/r02_launches_cfg2.csv python bench.py --config cfg2 --warmup 0 --steps 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_launches_cfg2.out 2>&1; echo "ncu exit $?"
ls -la gpurun_out/r02_launches_cfg2.csv; wc -l gpurun_out/r02_launches_cfg2.csv
