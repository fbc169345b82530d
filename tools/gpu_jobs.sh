#!/bin/bash
# The GPU jobs whose outputs are under profiles/ (run through gpurun on a B200, from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 2700 -- 'bash tools/gpu_jobs.sh <job> [<job> ...]'
# Outputs land in gpurun_out/ (scratch); the summaries worth keeping are copied into profiles/.
#   tests      the whole -m gpu suite
#   bench      default bench line (cfg3, with e2e and cpu_baseline)
#   timeline   cfg3 bench with the per-launch profile -> critical-path timeline + class summary
#   cfg4       cfg4 bench line
#   dist1      the multi-GPU path at N = 1 through NCCL (--force-dist)
#   launches   ncu launch list of the bench command (cfg2) -> launch summary
#   ncu_gemm   ncu --set full of the long-K sketch GEMM at cfg3 shape
#   panel      panel-QR latency per algorithm + per-launch breakdown + CholeskyQR2 phase clocks
#   scaling    per-rank replay of lstsq_dist at cfg3, P = 1, 2, 4, 8 + the scaling model
#   sanitize   compute-sanitizer memcheck / racecheck / synccheck / initcheck (tools/sanitize_all.sh)
cd "${GRAFT_REPO_ROOT:-.}" || exit 1
mkdir -p gpurun_out
summ() { python - "$@" <<'PY'
import json, sys
for f in sys.argv[1:]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["time_to_solution_s"], d["value"], d["roofline"]["frac"], d.get("e2e", {}).get("seconds"))
PY
}
for job in "$@"; do
  case "$job" in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/pytest_gpu.log ;;
    bench) timeout 1500 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "bench exit $?"; summ gpurun_out/bench_cfg3.json ;;
    timeline) timeout 1200 python bench.py --no-cpu-baseline --no-e2e --profile-dump gpurun_out/prof_cfg3.csv > gpurun_out/bench_prof.json 2>/dev/null; echo "timeline bench exit $?"
      python tools/prof_summary.py gpurun_out/prof_cfg3.csv > gpurun_out/prof_cfg3_summary.txt
      python tools/timeline.py gpurun_out/prof_cfg3.csv > gpurun_out/timeline_cfg3.txt 2>&1; gzip -f gpurun_out/prof_cfg3.csv; head -14 gpurun_out/timeline_cfg3.txt ;;
    cfg4) timeout 1200 python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 exit $?"; summ gpurun_out/bench_cfg4.json ;;
    dist1) timeout 1200 python bench.py --force-dist --no-cpu-baseline --no-e2e > gpurun_out/bench_dist_n1.json 2> gpurun_out/bench_dist_n1.err; echo "dist1 exit $?"; summ gpurun_out/bench_dist_n1.json ;;
    launches) timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 9000 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --config cfg2 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1; echo "launches exit $?"
      python tools/ncu_launch_summary.py gpurun_out/launches_cfg2.csv > gpurun_out/launches_cfg2_summary.txt; gzip -f gpurun_out/launches_cfg2.csv ;;
    ncu_gemm) timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma -c 2 -o gpurun_out/ncu_gemm -f python tools/ncu_gemm.py 50000 > gpurun_out/ncu_gemm.log 2>&1; echo "ncu_gemm exit $?" ;;
    panel) timeout 300 python tools/panel_bench.py > gpurun_out/panel_bench.log 2>&1; echo "panel exit $?"; grep hqr gpurun_out/panel_bench.log | tr '\n' ' '; echo
      timeout 300 python tools/panel_breakdown.py 50000x256 200000x256 > gpurun_out/panel_breakdown.log 2>&1
      UTV_TRACE=1 python -m paper_2408_05238_b200.build --force > /dev/null 2>&1 && python tools/cqr_trace.py > gpurun_out/cqr_trace.log 2>&1
      python -m paper_2408_05238_b200.build --force > /dev/null 2>&1 ;;
    scaling) timeout 1500 python tools/dist_replay.py --n 50000 --b 256 --q 2 --k 1 --P 1 2 4 8 --out gpurun_out/dist_replay_cfg3.json > gpurun_out/dist_replay.log 2>&1; echo "replay exit $?"
      for bw in 400 600 800; do python tools/scaling_model.py gpurun_out/dist_replay_cfg3.json --busbw $bw --out gpurun_out/model_cfg3_busbw$bw.json > gpurun_out/model_cfg3_busbw$bw.txt 2>&1; done
      cat gpurun_out/model_cfg3_busbw600.txt; gzip -f gpurun_out/dist_replay_cfg3.json ;;
    sanitize) bash tools/sanitize_all.sh ;;
    *) echo "unknown job $job" ;;
  esac
done
