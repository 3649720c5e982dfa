"""One launch each of our tcgen05 GEMM and cuBLAS (torch.matmul) on the MLP-up shape, for ncu."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_02921_b200 import _lib
M, N, K = 65536, 16384, 4096
A = (torch.randn(M, K, device="cuda") * 0.5).half()
B = (torch.randn(N, K, device="cuda") * 0.02).half()
out = torch.empty(M, N, device="cuda", dtype=torch.float16)
s = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    _lib.check(_lib.lib().krr_gemm(_lib.GEMM_TCGEN05, _lib.F16, A.data_ptr(), B.data_ptr(), M, N, K,
                                   _lib.EPI_STORE, out.data_ptr(), None, s))
    torch.matmul(A, B.T, out=out)
torch.cuda.synchronize()
