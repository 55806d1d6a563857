for v in wait10000000 wait20000 wait1000; do
BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/b27_$v.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/b27_$v.json')); print('$v', d['ms_per_step'], d['value'], d['dense_ms_per_step'], d['dense_tflops'], d['speedup_vs_dense'])"
done
