"""One MLP-up GEMM launch at the C3 shape (M=307,200, N=16,384, K=4,096, GELU)
for DRAM-traffic capture under ncu (env: M rows, EPI = gelu | store | residual)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_02921_b200 import _lib
M, N, K = int(os.environ.get("M", 307200)), 16384, 4096
EPI = {"gelu": _lib.EPI_GELU, "store": _lib.EPI_STORE, "residual": _lib.EPI_RESIDUAL}[
    os.environ.get("EPI", "gelu")]
A = (torch.randn(M, K, device="cuda") * 0.5).half()
B = (torch.randn(N, K, device="cuda") * 0.02).half()
out = torch.empty(M, N, device="cuda", dtype=torch.float32 if EPI == _lib.EPI_RESIDUAL
                  else torch.float16)
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    _lib.check(_lib.lib().krr_gemm(_lib.GEMM_TCGEN05, _lib.F16, A.data_ptr(), B.data_ptr(), M, N,
                                   K, EPI, out.data_ptr(), None, s))
torch.cuda.synchronize()
