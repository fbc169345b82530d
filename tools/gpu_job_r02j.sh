cd $GRAFT_REPO_ROOT
UTV_TRACE=1 python -c 'from paper_2408_05238_b200 import build as b; b.build(force=True)' > /dev/null 2>&1
python tools/qr_phase_trace.py 200000
python tools/qr_phase_trace.py 101000
python tools/qr_phase_trace.py 150000
