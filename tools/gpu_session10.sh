set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -15
for m in 0 1 2; do
BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_emu$m.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench10_emu$m.json 2> gpurun_out/bench10_emu$m.err; tail -2 gpurun_out/bench10_emu$m.err; python -c "import json; d=json.load(open('gpurun_out/bench10_emu$m.json')); print('emu$m', d['ms_per_step'], d['value'], d['dense_ms_per_step'], d['dense_tflops'], d['speedup_vs_dense'])"
done
BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_emu2.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
