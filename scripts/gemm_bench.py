"""Micro-benchmark of the tcgen05 GEMM on the C3 (7B) shapes, per epilogue.

    python scripts/gemm_bench.py [--m 65536] [--reps 20]   (KRR_LIB=<variant .so> to A/B a variant library)

Prints TF/s per shape plus SM clock / power sampled during the loop, and
torch.matmul (cuBLAS) on the same shape for reference.
"""

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import tempfile
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_02921_b200 import _lib  # noqa: E402


def sample_clocks(fn):
    f = tempfile.NamedTemporaryFile("w+", delete=False)
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=f)
    try:
        out = fn()
    finally:
        p.terminate()
        p.wait()
    vals = [l.split(",") for l in open(f.name).read().strip().splitlines() if "," in l]
    sm = sorted(float(a) for a, _ in vals) or [0]
    pw = sorted(float(b) for _, b in vals) or [0]
    return out, sm[len(sm) // 2], pw[len(pw) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=65536)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    M = args.m
    d, hq, nqkv = 4096, 4096, 6144
    shapes = [("qkv", nqkv, d, _lib.EPI_STORE), ("wo", d, hq, _lib.EPI_RESIDUAL),
              ("up_gelu", 4 * d, d, _lib.EPI_GELU), ("down", d, 4 * d, _lib.EPI_RESIDUAL),
              ("up_store", 4 * d, d, _lib.EPI_STORE)]
    L = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    res = {"lib": os.environ.get("KRR_LIB", "default"), "M": M}
    for name, N, K, epi in shapes:
        A = (torch.randn(M, K, device="cuda") * 0.5).half()
        B = (torch.randn(N, K, device="cuda") * 0.02).half()
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == _lib.EPI_RESIDUAL
                          else torch.float16)

        def run():
            for _ in range(3):
                _lib.check(L.krr_gemm(_lib.GEMM_TCGEN05, _lib.F16, A.data_ptr(), B.data_ptr(), M,
                                      N, K, epi, out.data_ptr(), None, s))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(args.reps):
                _lib.check(L.krr_gemm(_lib.GEMM_TCGEN05, _lib.F16, A.data_ptr(), B.data_ptr(), M,
                                      N, K, epi, out.data_ptr(), None, s))
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / args.reps
        ms, mhz, watts = sample_clocks(run)
        tf = 2 * M * N * K / ms / 1e9
        res[name] = {"ms": round(ms, 3), "tflops": round(tf, 1), "sm_mhz": mhz, "watts": watts,
                     "flops_per_clk_sm": round(tf * 1e12 / (148 * mhz * 1e6)) if mhz else None}

        def run_cublas():
            for _ in range(3):
                torch.matmul(A, B.T)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(args.reps):
                torch.matmul(A, B.T)
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / args.reps
        if name in ("qkv", "up_store", "down"):
            ms, mhz, watts = sample_clocks(run_cublas)
            tf = 2 * M * N * K / ms / 1e9
            res[name + "_cublas"] = {"ms": round(ms, 3), "tflops": round(tf, 1), "sm_mhz": mhz,
                                     "watts": watts}
        del A, B, out
    print(json.dumps(res))


if __name__ == "__main__":
    main()
