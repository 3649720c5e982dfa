"""Attention kernel micro-benchmark (CUDA events, warm): the tcgen05 kernel over
16-bit prefix pages and over HRKV INT8/INT4 code pages (dequantised in-kernel).

    python scripts/attn_bench.py [--pairs 800] [--P 512] [--T 48] [--bits 16,8,4]
                                 [--boost 1 8] [--docs 0]

Random q/K/V with logit std ~ boost*1 (boost 8-16 mimics the unscaled random-init
model); reports ms per launch, achieved prefix-KV GB/s (bytes read per launch at the
page format) and attention TF/s.  --expand also times krr_dequant_pages of the same
pages (the separate expand pass the fused kernel replaces).
"""

import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_02921_b200 import _lib  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=800)
    ap.add_argument("--P", type=int, default=512)
    ap.add_argument("--T", type=int, default=48)
    ap.add_argument("--boost", type=float, nargs="+", default=[1.0, 8.0])
    ap.add_argument("--bits", default="16")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--expand", action="store_true")
    ap.add_argument("--docs", type=int, default=0, help="distinct prefix docs (0 = one per pair)")
    a = ap.parse_args()
    n, KVH, G, HD, T, P, L = a.pairs, 8, 4, 128, a.T, a.P, 2
    nd = a.docs or n
    sc = 1.0 / math.sqrt(math.sqrt(HD))
    pre = (torch.randn(nd, L, 2, KVH, P, HD, device="cuda") * sc).half()
    cur = (torch.randn(n, 1, 2, KVH, T, HD, device="cuda") * sc).half()
    es = 2
    doc_of = torch.arange(n, device="cuda", dtype=torch.int64) % nd
    cptr = torch.arange(n, device="cuda", dtype=torch.int64) * (cur[0].numel() * es) + cur.data_ptr()
    vlen = torch.full((n,), P, dtype=torch.int32, device="cuda")
    tv = torch.ones(n, T, dtype=torch.uint8, device="cuda")
    out = torch.empty(n * T, KVH * G * HD, dtype=torch.float16, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    flops = 4.0 * n * KVH * G * HD * (T * P + T * (T + 1) / 2)
    n_t = nd * L * 2
    for bits in [int(b) for b in a.bits.split(",")]:
        if bits == 16:
            base, nbytes, scales, page = pre, pre.numel() * es, None, pre[0].numel() * es
        else:
            tb = KVH * P * HD * bits // 8
            base = torch.empty(n_t * tb, dtype=torch.uint8, device="cuda")
            scales = torch.empty(n_t * KVH * HD, dtype=torch.float32, device="cuda")
            _lib.check(_lib.lib().krr_quant_pages(pre.data_ptr(), _lib.F16, n_t, KVH, P, HD, bits,
                                                  base.data_ptr(), scales.data_ptr(), s))
            nbytes, page = base.numel(), L * 2 * tb
        pptr = doc_of * page + base.data_ptr()
        kv_bytes = n * KVH * 2 * P * HD * bits / 8
        for boost in a.boost:
            q = (torch.randn(n * KVH, G * T, HD, device="cuda") * sc * boost).half()

            def run():
                _lib.check(_lib.lib().krr_attention_quant(
                    _lib.ATTN_TCGEN05, _lib.F16, q.data_ptr(), n, KVH, G, HD, T, P, 1, 0,
                    pptr.data_ptr(), vlen.data_ptr(), cptr.data_ptr(), tv.data_ptr(),
                    out.data_ptr(), base.data_ptr(), nbytes, cur.data_ptr(), cur.numel() * es,
                    bits, 0 if scales is None else scales.data_ptr(), s))
            ms = timed(run, a.reps)
            print(f"bits {bits:2d} boost {boost:5.1f} P {P} T {T} pairs {n}: {ms:8.3f} ms  "
                  f"prefix KV {kv_bytes / ms / 1e6:7.0f} GB/s  {flops / ms / 1e9:6.0f} TF/s  "
                  f"finite={bool(torch.isfinite(out).all())}", flush=True)
        if a.expand and bits < 16:
            dst = torch.empty_like(pre)

            def exp():
                _lib.check(_lib.lib().krr_dequant_pages(base.data_ptr(), scales.data_ptr(), bits,
                                                        n_t, KVH, P, HD, _lib.F16,
                                                        dst.data_ptr(), s))
            ms = timed(exp, a.reps)
            print(f"bits {bits:2d} expand pass (1 layer of {nd} docs' pages x L={L}): {ms:8.3f} ms")


if __name__ == "__main__":
    main()
