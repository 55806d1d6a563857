timeout 600 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -25
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench19.json 2> gpurun_out/bench19.err; tail -3 gpurun_out/bench19.err; python -c "import json; d=json.load(open('gpurun_out/bench19.json')); print('new', d['ms_per_step'], d['value'], d['dense_ms_per_step'], d['dense_tflops'], d['speedup_vs_dense'], d['skip_frac'], d['v_tiles_skipped_frac'])"
BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_trace.so timeout 300 python tools/trace_timeline.py 2>&1 | tail -40
