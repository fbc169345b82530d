#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py's cases (one process per tool x case).
#   TOOLS="racecheck" CASES="lstsq wide" bash tools/sanitize_all.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/san
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  for c in ${CASES:-lstsq lstsq256 qrglobal gemm wide ooc cholqr}; do
    timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_run.py $c > gpurun_out/san/${tool}_${c}.log 2>&1
    echo "$tool $c exit $?" | tee -a gpurun_out/san/summary.txt
  done
done
