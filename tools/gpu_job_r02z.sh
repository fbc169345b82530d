cd $GRAFT_REPO_ROOT
python tools/gemm_sizes.py 50000 30000 20000 10000 > gpurun_out/gemm_sizes_r02z.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dgemm_tma -c 2 -o gpurun_out/r02_ncu_gemm_nn -f python tools/ncu_gemm.py 50000 nn,tn > gpurun_out/ncu_nn.log 2>&1
ncu -i gpurun_out/r02_ncu_gemm_nn.ncu-rep --page raw --csv > gpurun_out/r02_ncu_gemm_nn_raw.csv
ncu -i gpurun_out/r02_ncu_gemm_nn.ncu-rep --page source --csv --print-source sass -k regex:dgemm > gpurun_out/r02_ncu_gemm_nn_src.csv 2>/dev/null
echo done
