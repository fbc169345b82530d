cd $GRAFT_REPO_ROOT
timeout 300 python tools/panel_bench.py > gpurun_out/panel_bench_m.txt 2>&1; cat gpurun_out/panel_bench_m.txt
timeout 1500 python bench.py > gpurun_out/bench_r02_final_cfg3.json 2> gpurun_out/bench_r02_final_cfg3.err; echo "bench exit $?"
timeout 1200 python bench.py --force-dist --no-cpu-baseline --no-e2e > gpurun_out/bench_r02_dist_n1.json 2> gpurun_out/bench_r02_dist_n1.err; echo "dist bench exit $?"
python - <<'PY'
import json
for f in ["gpurun_out/bench_r02_final_cfg3.json", "gpurun_out/bench_r02_dist_n1.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["value"], d["roofline"]["frac"], d.get("e2e", {}).get("seconds"), d.get("solution"))
    except Exception as e:
        print(f, "ERR", e)
PY
