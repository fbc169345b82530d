cd $GRAFT_REPO_ROOT
timeout 1200 python bench.py --no-cpu-baseline --no-e2e --profile-dump gpurun_out/prof_cfg3_r02.csv > gpurun_out/bench_prof.json 2>/dev/null; echo "bench exit $?"
python tools/prof_summary.py gpurun_out/prof_cfg3_r02.csv > gpurun_out/prof_cfg3_r02_summary.txt
python tools/timeline.py gpurun_out/prof_cfg3_r02.csv > gpurun_out/timeline_cfg3_r02.txt 2>&1
gzip -f gpurun_out/prof_cfg3_r02.csv
