timeout 600 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -15
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/b33.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/b33.json')); print('gs', d['ms_per_step'], d['value'], d['dense_ms_per_step'], d['dense_tflops'], d['speedup_vs_dense'])"
