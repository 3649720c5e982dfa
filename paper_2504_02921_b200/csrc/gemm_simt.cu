// CUDA-core GEMM (fp32 accumulate) — the fp32 "debug build" of the linear
// layers (tcgen05 has no fp32-operand kind).  Same epilogues and the same
// batch-invariant K order as the tcgen05 kernel.  Also accepts 16-bit
// operands so it can cross-check the tensor-core kernel on the device.
#include "epilogue.cuh"

namespace krr {
namespace simt {

constexpr int TM = 64, TN = 64, TK = 16, THREADS = 256;

template <typename T>
__global__ void __launch_bounds__(THREADS)
    gemm_simt_kernel(const T* __restrict__ A, const T* __restrict__ B, int64_t M, int N, int K,
                EpiParams ep) {
  __shared__ float sA[TK][TM + 4];
  __shared__ float sB[TK][TN + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * TM;
  const int n0 = blockIdx.x * TN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    // 64x16 tiles of A and B: 1024 elements each, 4 per thread
    for (int i = threadIdx.x; i < TM * TK; i += THREADS) {
      const int r = i / TK, c = i % TK;
      const int64_t gr = m0 + r;
      const int gk = k0 + c;
      sA[c][r] = (gr < M && gk < K) ? Act<T>::to(A[gr * K + gk]) : 0.f;
      const int gn = n0 + r;
      sB[c][r] = (gn < N && gk < K) ? Act<T>::to(B[(int64_t)gn * K + gk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < TK; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  if (ep.kind == KRR_EPI_GLU_GELU || ep.kind == KRR_EPI_GLU_SILU) {
    // the 64-column tile is one (gate 32 | up 32) block pair: gate threads
    // (tx < 8) publish act(gate) through shared memory, up threads combine
    __shared__ float sG[TM][33];
    const bool gelu = ep.kind == KRR_EPI_GLU_GELU;
    if (tx < 8) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float g = acc[i][j];
          sG[ty * 4 + i][tx * 4 + j] = gelu ? gelu_tanh(g) : g / (1.0f + expf(-g));
        }
    }
    __syncthreads();
    if (tx >= 8) {
      const int oc = n0 / 2 + (tx - 8) * 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t row = m0 + ty * 4 + i;
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = sG[ty * 4 + i][(tx - 8) * 4 + j] * acc[i][j];
        if (row < M) epi_apply<T>(ep, row, oc, v, 4);
      }
    }
    return;
  }
  const int col0 = n0 + tx * 4;
  if (col0 >= N) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = m0 + ty * 4 + i;
    if (row < M) epi_apply<T>(ep, row, col0, acc[i], min(4, N - col0));
  }
}

}  // namespace simt

int launch_gemm_simt(int act_dtype, const void* A, const void* B, int64_t M, int N, int K,
                     const EpiParams& ep, cudaStream_t s) {
  using namespace simt;
  KRR_REQUIRE(N % 2 == 0, KRR_ESHAPE, "SIMT GEMM needs even N");
  KRR_REQUIRE((ep.kind != KRR_EPI_GLU_GELU && ep.kind != KRR_EPI_GLU_SILU) || N % 64 == 0,
              KRR_ESHAPE, "gated-MLP GEMM needs N % 64 == 0");
  KRR_REQUIRE((M + TM - 1) / TM < 65535, KRR_ESHAPE, "SIMT GEMM: M too large for one launch");
  dim3 grid((N + TN - 1) / TN, (unsigned)((M + TM - 1) / TM));
  if (act_dtype == KRR_F32)
    gemm_simt_kernel<float><<<grid, THREADS, 0, s>>>((const float*)A, (const float*)B, M, N, K, ep);
  else if (act_dtype == KRR_F16)
    gemm_simt_kernel<__half><<<grid, THREADS, 0, s>>>((const __half*)A, (const __half*)B, M, N, K, ep);
  else
    gemm_simt_kernel<__nv_bfloat16><<<grid, THREADS, 0, s>>>((const __nv_bfloat16*)A,
                                                        (const __nv_bfloat16*)B, M, N, K, ep);
  return check_launch("gemm_simt");
}

}  // namespace krr
