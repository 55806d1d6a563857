timeout 300 python tools/trace_timeline.py 2>&1 | tail -60
