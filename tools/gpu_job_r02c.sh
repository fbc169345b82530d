cd $GRAFT_REPO_ROOT
UTV_TRACE=1 python -c 'from paper_2408_05238_b200 import build as b; b.build(force=True)' > /dev/null 2>&1
for m in 50000 20000 200000; do python tools/qr_phase_trace.py $m; done
