cd $GRAFT_REPO_ROOT
rm -f gpurun_out/san/summary.txt
TOOLS="memcheck racecheck synccheck" CASES="distooc" SAN_TIMEOUT=900 bash tools/sanitize_all.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qr2_kernel -s 2 -c 1 -o gpurun_out/r02_ncu_qr2 -f python tools/ncu_qr.py > gpurun_out/ncu_qr2.log 2>&1; echo "ncu qr2 exit $?"
ncu -i gpurun_out/r02_ncu_qr2.ncu-rep --page raw --csv > gpurun_out/r02_ncu_qr2_raw.csv 2>/dev/null
ncu -i gpurun_out/r02_ncu_qr2.ncu-rep --page details --csv > gpurun_out/r02_ncu_qr2_details.csv 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:jacobi_kernel -s 1 -c 1 -o gpurun_out/r02_ncu_jac -f python tools/ncu_jac.py > gpurun_out/ncu_jac.log 2>&1; echo "ncu jac exit $?"
ncu -i gpurun_out/r02_ncu_jac.ncu-rep --page raw --csv > gpurun_out/r02_ncu_jac_raw.csv 2>/dev/null
ncu -i gpurun_out/r02_ncu_jac.ncu-rep --page details --csv > gpurun_out/r02_ncu_jac_details.csv 2>/dev/null
ls -la gpurun_out | tail -12
