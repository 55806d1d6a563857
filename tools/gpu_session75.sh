# head pairs (default) vs query-block pairs for every group, alternating, l32k and l128k
V=$PWD/paper_2512_07011_b200/_lib/variants
for c in l32k l128k; do
for i in 1 2 3; do
  for t in default bpall; do
    if [ $t = default ]; then unset BSFA_LIB_PATH; else export BSFA_LIB_PATH=$V/libbsfa_b200_$t.so; fi
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$t', round(d['ms_per_step'],3), round(d['dense_ms_per_step'],3), round(d['speedup_vs_dense'],3), d['clocks']['sm_mhz'])"
  done
done
done
