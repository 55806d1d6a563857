timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -15
timeout 300 python tools/trace_timeline.py 2>&1 | grep -E "^(bsfa|dense) "
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench14.json 2> gpurun_out/bench14.err; tail -2 gpurun_out/bench14.err; python -c "import json; d=json.load(open('gpurun_out/bench14.json')); print('kt64', d['ms_per_step'], d['value'], d['dense_ms_per_step'], d['dense_tflops'], d['speedup_vs_dense'])"
