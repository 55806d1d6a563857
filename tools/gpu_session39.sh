export BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_tpr2.so
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -4
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b39.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/b39.json')); print('tpr2', round(d['ms_per_step'],3), round(d['value'],1), round(d['dense_ms_per_step'],3), round(d['dense_tflops'],1), round(d['speedup_vs_dense'],3))"
unset BSFA_LIB_PATH
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b39d.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/b39d.json')); print('tpr1', round(d['ms_per_step'],3), round(d['value'],1), round(d['dense_ms_per_step'],3), round(d['dense_tflops'],1), round(d['speedup_vs_dense'],3))"
export BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_tpr2.so
done
