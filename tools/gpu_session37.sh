for v in default emu2 emu0 nochain; do
if [ $v = default ]; then unset BSFA_LIB_PATH; else export BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_$v.so; fi
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b37_$v.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/b37_$v.json')); print('$v', round(d['ms_per_step'],3), round(d['value'],1), round(d['dense_ms_per_step'],3), round(d['dense_tflops'],1), round(d['speedup_vs_dense'],3))"
done
