for v in emu0 emu2; do
BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench21_$v.json 2> gpurun_out/bench21_$v.err; tail -2 gpurun_out/bench21_$v.err; python -c "import json; d=json.load(open('gpurun_out/bench21_$v.json')); print('$v', d['ms_per_step'], d['value'], d['dense_ms_per_step'], d['dense_tflops'], d['speedup_vs_dense'])"
done
BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_trace_emu0.so timeout 300 python tools/trace_timeline.py 2>&1 | grep -E "^(bsfa|dense) "
