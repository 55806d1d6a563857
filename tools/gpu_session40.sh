for v in default k3v3; do
if [ $v = default ]; then unset BSFA_LIB_PATH; else export BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_$v.so; fi
timeout 600 python tools/sweep.py --seqs 32768 131072 --densities 0.5 --steps 5 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['seq_len'], d['gate'], round(d['ms'],2), round(d.get('tflops', d.get('exec_tflops',0)),1), d.get('speedup_vs_dense'))"
done
