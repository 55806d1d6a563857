"""External dense-attention context rows on the same box (no reference counterpart).

    python tools/dense_context.py [--seqs 32768 131072] [--steps 3]

Times dense causal GQA attention of the Llama-3.1-8B shape (32 q / 8 kv heads,
d = 128, bf16) with library kernels, next to this repo's own dense and BSFA
launches on identical inputs:
  * torch SDPA, cuDNN backend (K/V expanded to 32 heads if GQA is refused)
  * torch SDPA, flash backend (FlashAttention-2 code recompiled for sm_100)
  * flashinfer fmha_varlen (CUTLASS sm100a FMHA, JIT-built on first use)
One JSON line per (seq, kernel): ms, exact causal TFLOP/s (4*d*N(N+1)/2*Hq).
Failures are reported as lines with an "error" key, not raised.
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

HQ, HKV, D = 32, 8, 128


def timed(fn, steps, warmup, stream):
    _, tot = bench.time_steps(fn, steps, warmup, stream)
    return tot / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, nargs="+", default=[32768, 131072])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--skip", nargs="*", default=[])
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    from torch.nn.attention import SDPBackend, sdpa_kernel
    import torch.nn.functional as F

    for n in args.seqs:
        cfg = dict(heads_q=HQ, heads_kv=HKV, seq_len=n, head_dim=D)
        q, k, v = bench.make_inputs(cfg, 0, dev)
        flops = 4 * D * n * (n + 1) / 2 * HQ

        def report(name, fn, note=""):
            if name in args.skip:
                return
            try:
                t0 = time.perf_counter()
                fn()
                torch.cuda.synchronize()
                first = time.perf_counter() - t0
                ms = timed(fn, args.steps, 1, stream)
                print(json.dumps({"seq_len": n, "kernel": name, "ms": ms, "tflops_exact_causal": flops / ms / 1e9,
                                  "first_call_s": round(first, 2), "note": note}), flush=True)
            except Exception as e:  # context rows are best effort
                print(json.dumps({"seq_len": n, "kernel": name, "error": str(e).splitlines()[0][:300]}),
                      flush=True)
            torch.cuda.empty_cache()

        import paper_2512_07011_b200 as bsfa
        from paper_2512_07011_b200 import costs
        tiles = bsfa.TileConfig(128, 64)
        dplan = bsfa.BsfaPlan(1, HQ, HKV, n, D, tiles=tiles, device=dev)
        report("bsfa_b200_dense (this repo, DenseGate)", lambda: dplan.run(q, k, v))
        kl = costs.k_for_density(n, tiles, 0.5)
        thr = bench.calibrated_thresholds(cfg, tiles, kl, dev)
        plan = bsfa.BsfaPlan(1, HQ, HKV, n, D, tiles=tiles, thresholds=thr, k_level=kl, device=dev)
        report("bsfa_b200 threshold ~50% skip (this repo)", lambda: plan.run(q, k, v),
               "TFLOP/s column is dense-equivalent (exact causal flops / time)")
        del dplan, plan

        def sdpa(backend, gqa):
            if gqa:
                def f():
                    with sdpa_kernel(backend):
                        return F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
                return f
            ke = k.repeat_interleave(HQ // HKV, dim=1)
            ve = v.repeat_interleave(HQ // HKV, dim=1)

            def f():
                with sdpa_kernel(backend):
                    return F.scaled_dot_product_attention(q, ke, ve, is_causal=True)
            return f

        for name, be in (("torch_sdpa_cudnn", SDPBackend.CUDNN_ATTENTION), ("torch_sdpa_flash", SDPBackend.FLASH_ATTENTION)):
            try:
                fn = sdpa(be, True)
                fn()
                report(name, fn, "enable_gqa=True")
            except Exception:
                report(name, sdpa(be, False), "K/V expanded to 32 heads")

        def flashinfer_varlen():
            import flashinfer
            qn = q[0].transpose(0, 1).contiguous()  # [N, Hq, d]
            kn = k[0].transpose(0, 1).contiguous()
            vn = v[0].transpose(0, 1).contiguous()
            seg = torch.tensor([0, n], dtype=torch.int32, device=dev)
            return lambda: flashinfer.prefill.fmha_varlen(qn, kn, vn, seg, seg, max_qo_len=n, causal=True)

        if "flashinfer_fmha_varlen" not in args.skip:
            try:
                report("flashinfer_fmha_varlen (cutlass sm100a)", flashinfer_varlen())
            except Exception as e:
                print(json.dumps({"seq_len": n, "kernel": "flashinfer_fmha_varlen", "error": str(e)[:300]}))
        del q, k, v
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
