cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or scale or nullify or keep or wide or fullpath" > gpurun_out/pytest_aa.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/pytest_aa.log
timeout 900 python bench.py --no-cpu-baseline --profile-dump gpurun_out/prof_cfg3_aa.csv > gpurun_out/bench_aa.json 2>gpurun_out/bench_aa.err; echo "bench exit $?"
python tools/timeline.py gpurun_out/prof_cfg3_aa.csv > gpurun_out/timeline_cfg3_aa.txt 2>&1
gzip -f gpurun_out/prof_cfg3_aa.csv
python tools/jac_insitu.py cfg3 > gpurun_out/jac_insitu_aa.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_aa.json').read().strip().splitlines()[-1]); print(d['time_to_solution_s'], d['value'], d['roofline']['frac'], d['e2e'])"
head -16 gpurun_out/timeline_cfg3_aa.txt
