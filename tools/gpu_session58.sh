# CTA-pair kernel (BSFA_PAIR=1): first light -- a tiny GQA-4 case, then parity, then bench
export BSFA_LIB_PATH=$PWD/paper_2512_07011_b200/_lib/variants/libbsfa_b200_pair.so
timeout 300 python - <<'PY'
import numpy as np, torch, sys
sys.path.insert(0, ".")
import paper_2512_07011_b200 as bsfa
from oracle import bsfa_oracle as orc
torch.manual_seed(0)
for n, T in ((256, None), (1024, None), (1024, 3.6)):
    q = torch.randn(1, 4, n, 128, device="cuda").bfloat16(); k = torch.randn(1, 1, n, 128, device="cuda").bfloat16()
    v = torch.randn(1, 1, n, 128, device="cuda").bfloat16()
    if T is None:
        r = bsfa.attention(q, k, v)
        o = r.o.float().cpu().numpy()
        for h in range(4):
            ref, _ = orc.dense_attention(q[0, h].float().cpu().numpy(), k[0, 0].float().cpu().numpy(), v[0, 0].float().cpu().numpy(), True) if False else (None, None)
            ref = orc.dense_attention(q[0, h].float().cpu().numpy(), k[0, 0].float().cpu().numpy(), v[0, 0].float().cpu().numpy(), True)
            ref = ref[0] if isinstance(ref, tuple) else ref
            print("dense", n, h, float(np.abs(o[0, h] - ref).max()))
    else:
        t = bsfa.ThresholdTensor(values=np.full((1, 1, 4, n // 128), T, np.float32), k_levels=(1,), n_max=n, b_m=128, b_n=64)
        r = bsfa.attention(q, k, v, thresholds=t, k_level=1, return_trace=True)
        print("bsfa", n, "counters", r.counters.cpu().tolist(), "status", int(r.status.item()))
PY
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b58_pair.json 2>gpurun_out/b58_pair.err
python -c "import json; d=json.load(open('gpurun_out/b58_pair.json')); print('pair', round(d['ms_per_step'],3), round(d['value'],1), round(d['dense_ms_per_step'],3), round(d['dense_tflops'],1), round(d['speedup_vs_dense'],3))" || tail -3 gpurun_out/b58_pair.err
unset BSFA_LIB_PATH
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b58_def.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/b58_def.json')); print('default', round(d['ms_per_step'],3), round(d['value'],1), round(d['dense_ms_per_step'],3), round(d['dense_tflops'],1), round(d['speedup_vs_dense'],3))"
