// Prefix + causal-suffix attention (model.py:349-394, _exp_rows :406-436).
//
// Work unit = (sequence b, kv head).  Query rows are the G query heads of
// that kv head packed as row = g*T + t (model.py:377-378).  Keys are
//   [prefix: P cached positions, visible iff j < prefix_valid_len[b]]
//   [current: T positions, visible iff tok_valid[b,j] && j <= t]
// Logits are raw q.k (NO 1/sqrt(hd), model.py:380,383); the softmax max and
// sum are shared across both pieces; a row with no visible key outputs 0.
//
// Two kernels:
//   attn_mma   16-bit operands on mma.sync m16n8k16 tensor cores, fp32 online
//              softmax, cp.async double-buffered K/V blocks (the fast path).
//   attn_simt  fp32 CUDA-core two-pass softmax, op order of the reference
//              (the fp32 debug build used for the 1e-4 parity gate).
#include "launchers.h"
#include <math_constants.h>

namespace krr {

template <typename T>
__device__ __forceinline__ const T* kv_ptr(void* const* slabs, int b, int layer, int which,
                                           int KVH, int kvh, int len, int HD) {
  return reinterpret_cast<const T*>(slabs[b]) +
         ((int64_t)((layer * 2 + which) * KVH + kvh) * len) * HD;
}

// ============================================================ SIMT (fp32)
namespace attn_simt {
constexpr int WARPS = 4;

template <typename T>
__global__ void __launch_bounds__(WARPS * 32) attn_prefix_simt(AttnParams p) {
  extern __shared__ float sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = p.group, T_ = p.seq_len, P = p.prefix_len, HD = p.head_dim;
  const int KVH = p.kv_heads;
  const int nkeys = P + T_;
  float* logits = sm + warp * (nkeys + HD);
  float* qv = logits + nkeys;
  const int unit = blockIdx.y;
  const int b = unit / KVH, kvh = unit % KVH;
  const int row = blockIdx.x * WARPS + warp;
  if (row >= G * T_) return;
  const int g = row / T_, t = row % T_;
  const T* q = reinterpret_cast<const T*>(p.q) + ((int64_t)unit * G * T_ + row) * HD;
  for (int c = lane; c < HD; c += 32) qv[c] = Act<T>::to(q[c]);
  __syncwarp();
  const int vlen = P ? p.prefix_valid_len[b] : 0;
  const T* Kp = P ? kv_ptr<T>(p.prefix_kv, b, p.layer, 0, KVH, kvh, P, HD) : nullptr;
  const T* Vp = P ? kv_ptr<T>(p.prefix_kv, b, p.layer, 1, KVH, kvh, P, HD) : nullptr;
  const T* Kc = kv_ptr<T>(p.cur_kv, b, p.cur_layer, 0, KVH, kvh, T_, HD);
  const T* Vc = kv_ptr<T>(p.cur_kv, b, p.cur_layer, 1, KVH, kvh, T_, HD);
  const uint8_t* tv = p.tok_valid + (int64_t)b * T_;
  // logits (lane per key, ascending channel order)
  for (int j = lane; j < nkeys; j += 32) {
    bool vis;
    const T* kr;
    if (j < P) { vis = j < vlen; kr = Kp + (int64_t)j * HD; }
    else { const int jj = j - P; vis = tv[jj] && jj <= t; kr = Kc + (int64_t)jj * HD; }
    float s = -CUDART_INF_F;
    if (vis) {
      s = 0.f;
      for (int c = 0; c < HD; ++c) s = fmaf(qv[c], Act<T>::to(kr[c]), s);
    }
    logits[j] = s;
  }
  __syncwarp();
  float m = -CUDART_INF_F;
  for (int j = lane; j < nkeys; j += 32) m = fmaxf(m, logits[j]);
  m = warp_max(m);
  if (!isfinite(m)) m = 0.f;                       // model.py:425-426
  float z = 0.f;
  for (int j = lane; j < nkeys; j += 32) {
    const float e = expf(logits[j] - m);
    logits[j] = e;
    z += e;
  }
  z = warp_sum(z);
  if (z == 0.f) z = 1.f;                           // model.py:434-435
  __syncwarp();
  T* out = reinterpret_cast<T*>(p.out) + ((int64_t)b * T_ + t) * (KVH * G * HD) +
           (int64_t)(kvh * G + g) * HD;
  for (int c = lane; c < HD; c += 32) {
    float ac = 0.f, ap = 0.f;                      // current piece, then prefix piece (:391-393)
    for (int j = 0; j < T_; ++j) ac = fmaf(logits[P + j], Act<T>::to(Vc[(int64_t)j * HD + c]), ac);
    for (int j = 0; j < P; ++j) ap = fmaf(logits[j], Act<T>::to(Vp[(int64_t)j * HD + c]), ap);
    out[c] = Act<T>::from((ac + ap) / z);
  }
}
}  // namespace attn_simt

int launch_attention_simt(int act_dtype, const AttnParams& p, cudaStream_t s) {
  using namespace attn_simt;
  const int rows = p.group * p.seq_len;
  dim3 grid((rows + WARPS - 1) / WARPS, p.n_seqs * p.kv_heads);
  KRR_REQUIRE(grid.y < 65536, KRR_ESHAPE, "SIMT attention: too many units");
  const size_t smem = (size_t)WARPS * (p.prefix_len + p.seq_len + p.head_dim) * sizeof(float);
  KRR_REQUIRE(smem <= 200 * 1024, KRR_ESHAPE, "SIMT attention: sequence too long");
  if (act_dtype == KRR_F32) {
    cudaFuncSetAttribute(attn_prefix_simt<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_prefix_simt<float><<<grid, WARPS * 32, smem, s>>>(p);
  } else if (act_dtype == KRR_F16) {
    cudaFuncSetAttribute(attn_prefix_simt<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_prefix_simt<__half><<<grid, WARPS * 32, smem, s>>>(p);
  } else {
    cudaFuncSetAttribute(attn_prefix_simt<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_prefix_simt<__nv_bfloat16><<<grid, WARPS * 32, smem, s>>>(p);
  }
  return check_launch("attention_simt");
}

// ============================================================ mma.sync (16-bit)
namespace attn_mma {




__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void ldm_x4(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                       const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(su32(p)));
}
__device__ __forceinline__ void ldm_x4_t(uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                         const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(su32(p)));
}
template <typename T>
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  if constexpr (std::is_same<T, __half>::value) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
}
template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  if constexpr (std::is_same<T, __half>::value) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}


// One CTA per (sequence, kv head) unit — or per slice of its G*T rows when
// that exceeds max_warps*16 — so every K/V block is fetched into shared
// memory once and reused by all query rows of the unit (all G heads of the
// GQA group).  Warp w owns 16 rows.  K/V blocks of KB keys stream through a
// STAGES-deep cp.async ring; row pitch HD+8 elements (16 B pad) keeps
// ldmatrix conflict-free.
constexpr int STAGES = 3;

template <typename T, int HD, int KB>
__global__ void __launch_bounds__(384, 1) attn_prefix_mma(AttnParams p, int row_blocks) {
  constexpr int PITCH = HD + 8;
  constexpr int CPR = HD / 8;  // 16 B chunks per row
  extern __shared__ __align__(16) uint8_t smem[];
  const int nwarps = blockDim.x >> 5;
  const int rows_cta = nwarps * 16;
  T* sQ = reinterpret_cast<T*>(smem);
  T* sK = sQ + rows_cta * PITCH;                 // [STAGES][KB][PITCH]
  T* sV = sK + STAGES * KB * PITCH;              // [STAGES][KB][PITCH]
  uint8_t* sTV = reinterpret_cast<uint8_t*>(sV + STAGES * KB * PITCH);  // [T]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nthr = blockDim.x;
  const int G = p.group, T_ = p.seq_len, P = p.prefix_len, KVH = p.kv_heads;
  const int unit = blockIdx.x / row_blocks;
  const int rb = blockIdx.x - unit * row_blocks;
  const int b = unit / KVH, kvh = unit - b * KVH;
  const int row0 = rb * rows_cta;
  const int nrows = G * T_;

  const T* qg = reinterpret_cast<const T*>(p.q) + ((int64_t)unit * nrows) * HD;
  for (int i = threadIdx.x; i < rows_cta * CPR; i += nthr) {
    const int r = i / CPR, c = (i - r * CPR) * 8;
    const bool ok = row0 + r < nrows;
    cp_async16(sQ + r * PITCH + c, qg + (int64_t)(ok ? row0 + r : 0) * HD + c, ok);
  }
  for (int j = threadIdx.x; j < T_; j += nthr) sTV[j] = p.tok_valid[(int64_t)b * T_ + j];

  // key ranges: prefix [0, vlen), current [0, cur_end)
  const int vlen = P ? min(p.prefix_valid_len[b], P) : 0;
  const int last_row = min(row0 + rows_cta, nrows) - 1;
  const int t_max = (last_row / T_ != row0 / T_) ? T_ - 1 : last_row % T_;
  const int cur_end = t_max + 1;
  const int nb_pre = (vlen + KB - 1) / KB;
  const int nb_cur = (cur_end + KB - 1) / KB;
  const int nblocks = nb_pre + nb_cur;

  const T* Kp = P ? kv_ptr<T>(p.prefix_kv, b, p.layer, 0, KVH, kvh, P, HD) : nullptr;
  const T* Vp = P ? kv_ptr<T>(p.prefix_kv, b, p.layer, 1, KVH, kvh, P, HD) : nullptr;
  const T* Kc = kv_ptr<T>(p.cur_kv, b, p.cur_layer, 0, KVH, kvh, T_, HD);
  const T* Vc = kv_ptr<T>(p.cur_kv, b, p.cur_layer, 1, KVH, kvh, T_, HD);

  auto load_block = [&](int blk) {
    if (blk >= nblocks) return;
    const int buf = blk % STAGES;
    const bool pre = blk < nb_pre;
    const int k0 = pre ? blk * KB : (blk - nb_pre) * KB;
    const int lim = pre ? vlen : cur_end;
    const T* Ks = pre ? Kp : Kc;
    const T* Vs = pre ? Vp : Vc;
    T* dk = sK + buf * KB * PITCH;
    T* dv = sV + buf * KB * PITCH;
    for (int i = threadIdx.x; i < KB * CPR; i += nthr) {
      const int r = i / CPR, c = (i - r * CPR) * 8;
      const bool ok = k0 + r < lim;
      const int64_t off = (int64_t)(ok ? k0 + r : 0) * HD + c;
      cp_async16(dk + r * PITCH + c, Ks + off, ok);
      cp_async16(dv + r * PITCH + c, Vs + off, ok);
    }
  };

  // prologue: Q + blocks 0..STAGES-2, one commit group each
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    load_block(s);
    cp_commit();
  }

  const int r_lo = row0 + warp * 16 + (lane >> 2);
  const int r_hi = r_lo + 8;
  const int t_lo = r_lo % T_, t_hi = r_hi % T_;
  const bool warp_live = row0 + warp * 16 < nrows;
  float m_lo = -CUDART_INF_F, m_hi = -CUDART_INF_F, l_lo = 0.f, l_hi = 0.f;
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  const float L2E = 1.4426950408889634f;

  for (int blk = 0; blk < nblocks; ++blk) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    load_block(blk + STAGES - 1);
    cp_commit();
    if (!warp_live) continue;
    const int buf = blk % STAGES;
    const bool pre = blk < nb_pre;
    const int k0 = pre ? blk * KB : (blk - nb_pre) * KB;
    const T* cK = sK + buf * KB * PITCH;
    const T* cV = sV + buf * KB * PITCH;

    float s[KB / 8][4];
#pragma unroll
    for (int n = 0; n < KB / 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      uint32_t a[4];
      ldm_x4(a[0], a[1], a[2], a[3],
             sQ + (warp * 16 + (lane & 15)) * PITCH + kk * 16 + (lane >> 4) * 8);
#pragma unroll
      for (int n = 0; n < KB / 8; n += 2) {
        uint32_t b0, b1, b2, b3;
        const int kr = n * 8 + (lane & 7) + ((lane >> 4) << 3);
        const int kc = kk * 16 + ((lane >> 3) & 1) * 8;
        ldm_x4(b0, b1, b2, b3, cK + kr * PITCH + kc);
        mma16816<T>(s[n], a, b0, b1);
        mma16816<T>(s[n + 1], a, b2, b3);
      }
    }
    // mask + online softmax (shared max across prefix and current pieces)
    float mx_lo = -CUDART_INF_F, mx_hi = -CUDART_INF_F;
    const bool full_pre = pre && (k0 + KB <= vlen);
#pragma unroll
    for (int n = 0; n < KB / 8; ++n) {
      if (!full_pre) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int j = k0 + n * 8 + (lane & 3) * 2 + (e & 1);
          const int t = (e < 2) ? t_lo : t_hi;
          const bool vis = pre ? (j < vlen)
                               : ((j < T_) && (j <= t) && sTV[j < T_ ? j : 0]);
          if (!vis) s[n][e] = -CUDART_INF_F;
        }
      }
      mx_lo = fmaxf(mx_lo, fmaxf(s[n][0], s[n][1]));
      mx_hi = fmaxf(mx_hi, fmaxf(s[n][2], s[n][3]));
    }
    mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
    mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
    mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
    mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
    const float mn_lo = fmaxf(m_lo, mx_lo), mn_hi = fmaxf(m_hi, mx_hi);
    const float base_lo = (mn_lo == -CUDART_INF_F) ? 0.f : mn_lo * L2E;
    const float base_hi = (mn_hi == -CUDART_INF_F) ? 0.f : mn_hi * L2E;
    const float sc_lo = (m_lo == -CUDART_INF_F) ? 0.f : exp2f(m_lo * L2E - base_lo);
    const float sc_hi = (m_hi == -CUDART_INF_F) ? 0.f : exp2f(m_hi * L2E - base_hi);
    m_lo = mn_lo;
    m_hi = mn_hi;
    float rs_lo = 0.f, rs_hi = 0.f;
    uint32_t pf[KB / 16][4];
#pragma unroll
    for (int n = 0; n < KB / 8; ++n) {
      const float p0 = exp2f(fmaf(s[n][0], L2E, -base_lo));
      const float p1 = exp2f(fmaf(s[n][1], L2E, -base_lo));
      const float p2 = exp2f(fmaf(s[n][2], L2E, -base_hi));
      const float p3 = exp2f(fmaf(s[n][3], L2E, -base_hi));
      rs_lo += p0 + p1;
      rs_hi += p2 + p3;
      pf[n >> 1][(n & 1) * 2 + 0] = pack2<T>(p0, p1);
      pf[n >> 1][(n & 1) * 2 + 1] = pack2<T>(p2, p3);
    }
    l_lo = l_lo * sc_lo + rs_lo;
    l_hi = l_hi * sc_hi + rs_hi;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= sc_lo; o[i][1] *= sc_lo;
      o[i][2] *= sc_hi; o[i][3] *= sc_hi;
    }
#pragma unroll
    for (int kk = 0; kk < KB / 16; ++kk) {
      const uint32_t a[4] = {pf[kk][0], pf[kk][1], pf[kk][2], pf[kk][3]};
#pragma unroll
      for (int n = 0; n < HD / 8; n += 2) {
        uint32_t b0, b1, b2, b3;
        const int vr = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int vc = n * 8 + (lane >> 4) * 8;
        ldm_x4_t(b0, b1, b2, b3, cV + vr * PITCH + vc);
        mma16816<T>(o[n], a, b0, b1);
        mma16816<T>(o[n + 1], a, b2, b3);
      }
    }
  }
  cp_wait<0>();
  if (!warp_live) return;

  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);
  const float inv_lo = l_lo > 0.f ? 1.f / l_lo : 0.f;
  const float inv_hi = l_hi > 0.f ? 1.f / l_hi : 0.f;
  const int H = KVH * G;
  if (r_lo < nrows) {
    const int g = r_lo / T_;
    T* dst = reinterpret_cast<T*>(p.out) + ((int64_t)b * T_ + t_lo) * (H * HD) +
             (kvh * G + g) * HD + (lane & 3) * 2;
#pragma unroll
    for (int n = 0; n < HD / 8; ++n)
      *reinterpret_cast<uint32_t*>(dst + n * 8) = pack2<T>(o[n][0] * inv_lo, o[n][1] * inv_lo);
  }
  if (r_hi < nrows) {
    const int g = r_hi / T_;
    T* dst = reinterpret_cast<T*>(p.out) + ((int64_t)b * T_ + t_hi) * (H * HD) +
             (kvh * G + g) * HD + (lane & 3) * 2;
#pragma unroll
    for (int n = 0; n < HD / 8; ++n)
      *reinterpret_cast<uint32_t*>(dst + n * 8) = pack2<T>(o[n][2] * inv_hi, o[n][3] * inv_hi);
  }
}

template <typename T, int HD, int KB>
int launch(const AttnParams& p, cudaStream_t s, int max_warps) {
  constexpr int PITCH = HD + 8;
  const int rows = p.group * p.seq_len;
  int warps = std::min(max_warps, (rows + 15) / 16);
  const int row_blocks = (rows + warps * 16 - 1) / (warps * 16);
  warps = (rows + row_blocks * 16 - 1) / (row_blocks * 16);  // balance the slices
  const size_t smem = (size_t)(warps * 16 + 2 * STAGES * KB) * PITCH * sizeof(T) +
                      ((p.seq_len + 15) & ~15);
  KRR_REQUIRE(smem <= 227 * 1024, KRR_ESHAPE, "attention: sequence too long for smem");
  const int64_t grid = (int64_t)row_blocks * p.n_seqs * p.kv_heads;
  KRR_REQUIRE(grid < INT32_MAX, KRR_ESHAPE, "attention grid too large");
  cudaFuncSetAttribute(attn_prefix_mma<T, HD, KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  attn_prefix_mma<T, HD, KB><<<(unsigned)grid, warps * 32, smem, s>>>(p, row_blocks);
  return check_launch("attention_mma");
}

template <typename T>
int dispatch(const AttnParams& p, cudaStream_t s) {
  switch (p.head_dim) {
    case 64: return launch<T, 64, 64>(p, s, 12);
    case 128: return launch<T, 128, 64>(p, s, 12);
    case 256: return launch<T, 256, 32>(p, s, 8);
    default: return fail(KRR_EUNSUPPORTED, "tensor-core attention supports head_dim 64/128/256");
  }
}

}  // namespace attn_mma


int launch_attention_mma(int act_dtype, const AttnParams& p, cudaStream_t s) {
  if (act_dtype == KRR_F16) return attn_mma::dispatch<__half>(p, s);
  if (act_dtype == KRR_BF16) return attn_mma::dispatch<__nv_bfloat16>(p, s);
  return fail(KRR_EUNSUPPORTED, "tensor-core attention needs a 16-bit dtype");
}

}  // namespace krr
