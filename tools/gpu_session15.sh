timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -5
timeout 300 python tools/trace_timeline.py 2>&1 | tail -30
