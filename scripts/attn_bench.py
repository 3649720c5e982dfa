"""Attention kernel micro-benchmark on the C3 shape (CUDA events, warm).

    python scripts/attn_bench.py [--pairs 800] [--boost 1 8] [--backends mma,tc]

Random q/K/V with logit std ~ boost*1 (boost 8-16 mimics the unscaled random-init
model); reports ms per launch and achieved KV GB/s per backend.
"""

import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_02921_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=800)
    ap.add_argument("--P", type=int, default=512)
    ap.add_argument("--T", type=int, default=48)
    ap.add_argument("--boost", type=float, nargs="+", default=[1.0, 8.0])
    ap.add_argument("--backends", default="mma,tc")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--docs", type=int, default=0, help="distinct prefix docs (0 = one per pair)")
    a = ap.parse_args()
    n, KVH, G, HD, T, P, L = a.pairs, 8, 4, 128, a.T, a.P, 2
    sc = 1.0 / math.sqrt(math.sqrt(HD))
    pre = (torch.randn(n, L, 2, KVH, P, HD, device="cuda") * sc).half()
    cur = (torch.randn(n, 1, 2, KVH, T, HD, device="cuda") * sc).half()
    es = 2
    doc_of = torch.arange(n, device="cuda", dtype=torch.int64)
    if a.docs:
        doc_of = doc_of % a.docs
    pptr = doc_of * (pre[0].numel() * es) + pre.data_ptr()
    cptr = torch.arange(n, device="cuda", dtype=torch.int64) * (cur[0].numel() * es) + cur.data_ptr()
    vlen = torch.full((n,), P, dtype=torch.int32, device="cuda")
    tv = torch.ones(n, T, dtype=torch.uint8, device="cuda")
    out = torch.empty(n * T, KVH * G * HD, dtype=torch.float16, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    kv_bytes = n * KVH * 2 * (P + T) * HD * es
    # QK^T + PV over the visible keys (prefix + causal suffix)
    flops = 4.0 * n * KVH * G * HD * (T * P + T * (T + 1) / 2)
    names = {"mma": _lib.ATTN_MMA, "tc": _lib.ATTN_TCGEN05}
    for boost in a.boost:
        q = (torch.randn(n * KVH, G * T, HD, device="cuda") * sc * boost).half()
        for name in a.backends.split(","):
            be = names[name]

            def run():
                _lib.check(_lib.lib().krr_attention(
                    be, _lib.F16, q.data_ptr(), n, KVH, G, HD, T, P, 1, 0, pptr.data_ptr(),
                    vlen.data_ptr(), cptr.data_ptr(), tv.data_ptr(), out.data_ptr(),
                    pre.data_ptr(), pre.numel() * es, cur.data_ptr(), cur.numel() * es, s))
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            print(f"boost {boost:5.1f} {name:4s} {ms:8.3f} ms  KV {kv_bytes / ms / 1e6:7.0f} GB/s  "
                  f"{flops / ms / 1e9:6.0f} TF/s  "
                  f"finite={bool(torch.isfinite(out).all())}", flush=True)


if __name__ == "__main__":
    main()
