# CTA-pair kernel: st.async decisions, CTA-scope arrives -- parity + bench
V=$PWD/paper_2512_07011_b200/_lib/variants
export BSFA_LIB_PATH=$V/libbsfa_b200_split.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for i in 1 2; do
for t in split default; do
  if [ $t = default ]; then unset BSFA_LIB_PATH; else export BSFA_LIB_PATH=$V/libbsfa_b200_$t.so; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b66_$t.json 2>gpurun_out/b66_$t.err
  python -c "import json; d=json.load(open('gpurun_out/b66_$t.json')); print('$t', round(d['ms_per_step'],3), round(d['value'],1), round(d['dense_ms_per_step'],3), round(d['dense_tflops'],1), round(d['speedup_vs_dense'],3))" 2>/dev/null || echo "$t failed"
done
done
