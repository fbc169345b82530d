cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_cqr_all.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_cqr_all.log
timeout 900 python bench.py --no-cpu-baseline --profile-dump gpurun_out/prof_cfg3_cqr.csv > gpurun_out/bench_cfg3_cqr.json 2>gpurun_out/bench_cfg3_cqr.err; echo "bench3 exit $?"
python tools/timeline.py gpurun_out/prof_cfg3_cqr.csv > gpurun_out/timeline_cfg3_cqr.txt 2>&1; gzip -f gpurun_out/prof_cfg3_cqr.csv
timeout 900 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/bench_cfg4_cqr.json 2>gpurun_out/bench_cfg4_cqr.err; echo "bench4 exit $?"
for f in gpurun_out/bench_cfg3_cqr.json gpurun_out/bench_cfg4_cqr.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['time_to_solution_s'], d['value'], d['roofline']['frac'], d['hbm_kernels']['panel'])"; done
head -30 gpurun_out/timeline_cfg3_cqr.txt
