"""G=8 (CTA-pair, 256 rows per SM) GEMM check: run the same launches with
KRR_GEMM_PAIR=0 and =1 in two subprocesses and compare outputs bit for bit, plus
a fp32 torch reference.  The G=8 geometry is not in the tree: apply
scripts/variants/gemm_pair_g8.patch (KRR_GEMM_PAIR switch; -DEXP_NO_EPI gives the
timing-only no-epilogue build) and rebuild.  usage: python scripts/pair_check.py"""
import os, subprocess, sys
import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "run":
    import math, torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2504_02921_b200 import _lib
    torch.manual_seed(0)
    out = {}
    s = torch.cuda.current_stream().cuda_stream
    for (M, N, K) in [(65536 + 300, 768, 1024), (70000, 512, 4096), (20000, 1024, 384),
                      (17000, 256, 256)]:
        A = (torch.randn(M, K, device="cuda") * 0.5).half()
        B = (torch.randn(N, K, device="cuda") / math.sqrt(K)).half()
        for epi in (_lib.EPI_STORE, _lib.EPI_GELU, _lib.EPI_RESIDUAL):
            if epi == _lib.EPI_RESIDUAL:
                o = torch.randn(M, N, device="cuda")
            else:
                o = torch.empty(M, N, dtype=torch.float16, device="cuda")
            _lib.check(_lib.lib().krr_gemm(_lib.GEMM_TCGEN05, _lib.F16, A.data_ptr(), B.data_ptr(),
                                           M, N, K, epi, o.data_ptr(), None, s))
            torch.cuda.synchronize()
            out[f"{M}_{N}_{K}_{epi}"] = o.float().cpu().numpy()
        ref = (A.float() @ B.float().T).cpu().numpy()
        out[f"ref_{M}_{N}_{K}"] = ref
    np.savez(sys.argv[2], **out)
    sys.exit(0)

res = {}
for pair in ("0", "1"):
    f = f"/tmp/pair_{pair}.npz"
    env = dict(os.environ, KRR_GEMM_PAIR=pair)
    subprocess.run([sys.executable, __file__, "run", f], env=env, check=True)
    res[pair] = np.load(f)
for k in res["0"].files:
    if k.startswith("ref"):
        continue
    a, b = res["0"][k], res["1"][k]
    M, N, K, epi = k.split("_")
    ref = res["0"][f"ref_{M}_{N}_{K}"]
    note = ""
    if epi == "0":
        note = f"max|pair-ref| {np.abs(b - ref).max():.3e}"
    print(k, "bit-identical" if np.array_equal(a, b) else f"DIFF max {np.abs(a-b).max():.3e}", note)
