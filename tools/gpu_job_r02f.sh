cd $GRAFT_REPO_ROOT
timeout 1200 python bench.py > gpurun_out/bench_r02_cfg3.json 2> gpurun_out/bench_r02_cfg3.err; echo "bench exit $?"
tail -c 600 gpurun_out/bench_r02_cfg3.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma -c 2 -o gpurun_out/r02_ncu_gemm -f python tools/ncu_gemm.py 50000 > gpurun_out/ncu_gemm.log 2>&1; echo "ncu exit $?"
ncu -i gpurun_out/r02_ncu_gemm.ncu-rep --page raw --csv > gpurun_out/r02_ncu_gemm_raw.csv 2>/dev/null
ls -la gpurun_out/
