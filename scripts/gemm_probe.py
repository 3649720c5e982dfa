"""One tcgen05 GEMM shape in a sustained loop: TF/s, SM clock and board power
(nvidia-smi sampled during the loop).  Used for A/B of GEMM variants
(KRR_LIB=<variant .so>) and as the target of ncu captures.

    python scripts/gemm_probe.py [--shape up_store|up_gelu|down|qkv|wo] [--m 65536]
                                 [--reps 150] [--cublas]
"""

import argparse
import json
import os
import subprocess
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_02921_b200 import _lib  # noqa: E402

SHAPES = {"qkv": (6144, 4096, _lib.EPI_STORE), "wo": (4096, 4096, _lib.EPI_RESIDUAL),
          "up_gelu": (16384, 4096, _lib.EPI_GELU), "down": (4096, 16384, _lib.EPI_RESIDUAL),
          "up_store": (16384, 4096, _lib.EPI_STORE)}


def sampled(fn):
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
    ap.add_argument("--shape", default="up_store")
    ap.add_argument("--m", type=int, default=65536)
    ap.add_argument("--reps", type=int, default=150)
    ap.add_argument("--cublas", action="store_true")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    N, K, epi = SHAPES[a.shape]
    M = a.m
    A = (torch.randn(M, K, device="cuda") * 0.5).half()
    B = (torch.randn(N, K, device="cuda") * 0.02).half()
    out = torch.zeros(M, N, device="cuda",
                      dtype=torch.float32 if epi == _lib.EPI_RESIDUAL else torch.float16)
    L = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream

    def one():
        if a.cublas:
            torch.matmul(A, B.T, out=out) if out.dtype == torch.float16 else torch.matmul(A, B.T)
        else:
            _lib.check(L.krr_gemm(_lib.GEMM_TCGEN05, _lib.F16, A.data_ptr(), B.data_ptr(), M, N,
                                  K, epi, out.data_ptr(), None, s))

    def run():
        for _ in range(3):
            one()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(a.reps):
            one()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    ms, mhz, watts = sampled(run)
    tf = 2 * M * N * K / ms / 1e9
    print(json.dumps({"tag": a.tag, "lib": os.path.basename(_lib.LIB_PATH),
                      "mode": os.environ.get("KRR_GEMM_CTA", "default"), "shape": a.shape,
                      "M": M, "cublas": a.cublas, "ms": round(ms, 3), "tflops": round(tf, 1),
                      "sm_mhz": mhz, "watts": watts,
                      "tf_per_ghz": round(tf / (mhz / 1000), 1) if mhz else None}))


if __name__ == "__main__":
    main()
