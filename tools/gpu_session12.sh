timeout 300 python tools/trace_timeline.py 2>&1 | tail -30
BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_noturn.so timeout 300 python tools/trace_timeline.py 2>&1 | tail -30
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench12.json 2> gpurun_out/bench12.err; tail -2 gpurun_out/bench12.err; python -c "import json; d=json.load(open('gpurun_out/bench12.json')); print('default', d['ms_per_step'], d['value'], d['dense_ms_per_step'], d['dense_tflops'], d['speedup_vs_dense'])"
