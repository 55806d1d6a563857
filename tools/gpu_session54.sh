# compile-time gate mode (threshold) vs runtime gate mode: BSFA only, A/B x3
V=$PWD/paper_2512_07011_b200/_lib/variants
for i in 1 2 3; do
  for t in default fixed; do
    if [ $t = default ]; then unset BSFA_LIB_PATH; else export BSFA_LIB_PATH=$V/libbsfa_b200_$t.so; fi
    timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-dense > gpurun_out/b54_$t.json 2>gpurun_out/b54_$t.err
    python -c "import json; d=json.load(open('gpurun_out/b54_$t.json')); print('$t', round(d['ms_per_step'],3), round(d['value'],1))" || tail -3 gpurun_out/b54_$t.err
  done
done
