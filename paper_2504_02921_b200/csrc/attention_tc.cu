// Tensor-core prefix + causal-suffix attention for sm_100a (tcgen05 / TMEM / TMA).
//
// Semantics as attention.cu (model.py:349-394, _exp_rows :406-436): raw q.k
// logits (no 1/sqrt(hd)), prefix keys visible iff j < prefix_valid_len[b],
// current keys visible iff tok_valid[b,j] && j <= t, one softmax over both
// pieces, fully-masked rows output 0.
//
// CTA = (unit, 128-row tile); unit = (sequence b, kv head); tile rows are the
// GQA-packed query rows g*T+t of that unit (model.py:377-378), so every K/V
// block is fetched once for all G heads.  Two CTAs per SM (112 KB smem, 256
// TMEM columns each) so one CTA's prologue overlaps the other's work.
//
//   warp 0      TMA: Q tile once (2-D map over the packed q buffer); K and V
//               blocks of KB keys from the paged pool (3-D map [page][key][hd],
//               page = (slot, layer, K|V, kv_head)) into a 2-stage ring
//   warp 1      MMA (one thread): S = Q.K^T into TMEM (double-buffered, KB cols),
//               then O += P.V into TMEM (HD cols); V is the MN-major B operand
//   warps 2..5  softmax: tcgen05.ld a row of S per thread, mask, running max in
//               the log2 domain, P = exp2(s - m) -> 16-bit, 128B-swizzled into
//               smem (the A operand of P.V); O is rescaled in TMEM only when the
//               max grows by more than 2^8 (exact after the final 1/l)
//   epilogue    the softmax warps read O, scale by 1/l, write 16-bit rows of
//               the attention output [b*T+t][(kvh*G+g)*HD + c]
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math_constants.h>
#include <mutex>
#include "launchers.h"
#include "tc_ptx.cuh"

namespace krr {
namespace attn_tc {
using namespace tc;

constexpr int TM = 128;        // query rows per CTA = TMEM lanes
constexpr int STAGES = 2;      // K/V ring depth
constexpr int THREADS = 192;
constexpr float RESCALE_LOG2 = 15.0f;  // lazy O rescale threshold: P <= 2^15 < f16 max

struct Params {
  void* const* prefix_kv;
  const char* prefix_base;
  int64_t prefix_page_bytes;   // P*HD*elt
  void* const* cur_kv;
  const char* cur_base;
  int64_t cur_page_bytes;      // T*HD*elt
  const int32_t* prefix_valid_len;
  const uint8_t* tok_valid;
  void* out;
  int KVH, G, T, P, layer, cur_layer, R, row_tiles;
};

template <int HD, int KB>
struct Smem {
  static constexpr int ATOM = 128 * 128;               // 128 rows x 128 B (one swizzle column)
  static constexpr int Q_BYTES = (HD / 64) * TM * 128;
  static constexpr int KV_BYTES = (HD / 64) * KB * 128; // one of K or V per stage
  static constexpr int P_BYTES = (KB / 64) * TM * 128;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + Q_BYTES;
  static constexpr int V_OFF = K_OFF + STAGES * KV_BYTES;
  static constexpr int P_OFF = V_OFF + STAGES * KV_BYTES;
  static constexpr int BAR_OFF = P_OFF + P_BYTES;
  static constexpr int TOTAL = BAR_OFF + 128;
  // S: 2*KB, O: HD -> 256 columns (two CTAs per SM) up to HD=128, 512 for HD=256
  static constexpr int TMEM_COLS = (2 * KB + HD <= 256) ? 256 : 512;
  static_assert(2 * KB + HD <= TMEM_COLS, "TMEM budget");
};

template <typename T>
__device__ __forceinline__ uint32_t pack_2(float a, float b) {
  if constexpr (std::is_same<T, __half>::value) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}

template <typename T, int HD, int KB>
__global__ void __launch_bounds__(THREADS, 2)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                   const __grid_constant__ CUtensorMap tmPre,
                   const __grid_constant__ CUtensorMap tmCur, const Params p) {
  using S = Smem<HD, KB>;
  // No static smem and no over-alignment request: the dynamic window then
  // starts right after the 1 KB per-CTA reservation, i.e. 1024-aligned (checked
  // below), and two CTAs fit in the SM's 228 KB.
  extern __shared__ uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint8_t* sQ = smem + S::Q_OFF;
  uint8_t* sK = smem + S::K_OFF;
  uint8_t* sV = smem + S::V_OFF;
  uint8_t* sP = smem + S::P_OFF;
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;              // [STAGES]  K ring: freed when S = Q.K^T is done
  uint64_t* k_empty = k_full + STAGES;
  uint64_t* v_full = k_empty + STAGES;      // [STAGES]  V ring: freed when O += P.V is done
  uint64_t* v_empty = v_full + STAGES;
  uint64_t* s_full = v_empty + STAGES;      // [2]
  uint64_t* s_empty = s_full + 2;           // [2]
  uint64_t* p_full = s_empty + 2;
  uint64_t* pv_done = p_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x / p.row_tiles;
  const int rt = blockIdx.x - unit * p.row_tiles;
  const int b = unit / p.KVH, kvh = unit - b * p.KVH;
  const int T_ = p.T, R = p.R;
  const int row0 = rt * TM;
  const int last_row = min(row0 + TM, R) - 1;
  const int t_max = (last_row / T_ != row0 / T_) ? T_ - 1 : last_row % T_;
  const int vlen = p.P ? min(p.prefix_valid_len[b], p.P) : 0;
  const int nb_pre = (vlen + KB - 1) / KB;
  const int nb = nb_pre + (t_max + 1 + KB - 1) / KB;

  if (warp == 0 && lane == 0) {
    if ((smem_u32(smem) & 1023) != 0) __trap();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmPre)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmCur)) : "memory");
    mbar_init(q_full, 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) { mbar_init(&s_full[s], 1); mbar_init(&s_empty[s], 4); }
    mbar_init(p_full, 4);
    mbar_init(pv_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)), "n"(S::TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t O_COL = 2 * KB;

  if (warp == 0) {
    // lane 0 streams Q then K blocks, lane 1 streams V blocks: the K ring is
    // released as soon as S = Q.K^T completes, so K runs further ahead of the
    // softmax than V (which is held until O += P.V completes).
    if (lane < 2) {
      const bool is_k = lane == 0;
      if (is_k) {
        mbar_expect_tx(q_full, S::Q_BYTES);
#pragma unroll
        for (int a = 0; a < HD / 64; ++a)
          tma_load<1>(sQ + a * S::ATOM, &tmQ, smem_u32(q_full), a * 64, unit * R + row0);
      }
      const int pre_page = p.P ? (int)((reinterpret_cast<const char*>(p.prefix_kv[b]) -
                                        p.prefix_base) / p.prefix_page_bytes) +
                                     (p.layer * 2) * p.KVH + kvh
                               : 0;
      const int cur_page = (int)((reinterpret_cast<const char*>(p.cur_kv[b]) - p.cur_base) /
                                 p.cur_page_bytes) + (p.cur_layer * 2) * p.KVH + kvh;
      uint64_t* full = is_k ? k_full : v_full;
      uint64_t* empty = is_k ? k_empty : v_empty;
      uint8_t* ring = is_k ? sK : sV;
      const int vofs = is_k ? 0 : p.KVH;
      for (int j = 0; j < nb; ++j) {
        const int s = j % STAGES;
        mbar_wait(&empty[s], ((j / STAGES) & 1) ^ 1);
        mbar_expect_tx(&full[s], S::KV_BYTES);
        const bool pre = j < nb_pre;
        const CUtensorMap* map = pre ? &tmPre : &tmCur;
        const int key0 = (pre ? j : j - nb_pre) * KB;
        const int pk = (pre ? pre_page : cur_page) + vofs;
#pragma unroll
        for (int a = 0; a < HD / 64; ++a)
          tma_load3(ring + s * S::KV_BYTES + a * (KB * 128), map, &full[s], a * 64, key0, pk);
      }
    }
  } else if (warp == 1) {
    // whole warp walks the schedule, one elected lane issues the MMAs
    constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
    constexpr uint32_t idesc_s = (1u << 4) | (fmt << 7) | (fmt << 10) |
                                 ((uint32_t)(KB >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
    constexpr uint32_t idesc_o = (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 16) |
                                 ((uint32_t)(HD >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
    const uint64_t dQ = sw128_desc(smem_u32(sQ));
    const uint64_t dK = sw128_desc(smem_u32(sK));
    const uint64_t dP = sw128_desc(smem_u32(sP));
    const uint64_t dV = sw128_desc_mn(smem_u32(sV), KB * 128, 1024);
    mbar_wait(q_full, 0);
    for (int j = 0; j <= nb; ++j) {
      if (j < nb) {
        const int s = j % STAGES, sb = j & 1;
        mbar_wait(&k_full[s], (j / STAGES) & 1);
        mbar_wait(&s_empty[sb], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        if (elect_one_sync()) {
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            const uint32_t off = (k >> 2) * S::ATOM + (k & 3) * 32;
            const uint32_t koff = s * S::KV_BYTES + (k >> 2) * (KB * 128) + (k & 3) * 32;
            mma_f16<1>(tmem + sb * KB, dQ + (off >> 4), dK + (koff >> 4), idesc_s, k > 0);
          }
          mma_commit<1>(&k_empty[s]);
          mma_commit<1>(&s_full[sb]);
        }
        __syncwarp();
      }
      if (j >= 1) {
        const int jj = j - 1, s = jj % STAGES;
        mbar_wait(&v_full[s], (jj / STAGES) & 1);
        mbar_wait(p_full, jj & 1);
        tc_fence_after();
        if (elect_one_sync()) {
#pragma unroll
          for (int k = 0; k < KB / 16; ++k)
            mma_f16<1>(tmem + O_COL, dP + (((k >> 2) * S::ATOM + (k & 3) * 32) >> 4),
                       dV + ((s * S::KV_BYTES + k * 16 * 128) >> 4), idesc_o,
                       (jj > 0) || (k > 0));
          mma_commit<1>(&v_empty[s]);
          mma_commit<1>(pv_done);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------- softmax warps
    const int quad = warp & 3;
    const int lrow = quad * 32 + lane;
    const int r = row0 + lrow;
    const bool row_ok = r < R;
    const bool quad_live = row0 + quad * 32 < R;
    const int g = r / T_, t = r - g * T_;
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    const uint8_t* tv = p.tok_valid + (int64_t)b * T_;
    const float L2E = 1.4426950408889634f;
    float m_use = -CUDART_INF_F, l = 0.f;
    uint8_t* prow = sP + lrow * 128;
    const int sw = lrow & 7;

    for (int j = 0; j < nb; ++j) {
      const int sb = j & 1;
      mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      float sv[KB];
      if (quad_live) {
        uint32_t raw[KB / 32][32];
#pragma unroll
        for (int c = 0; c < KB / 32; ++c) tmem_ld32_nowait(lane_base + sb * KB + c * 32, raw[c]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < KB / 32; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(raw[c][i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);

      // Running max m (log2 units, i.e. of s*log2e) is only raised when the
      // block max exceeds it by 2^8, so O is rarely touched; P = 2^(s*log2e - m)
      // <= 256 fits the 16-bit operand.  Masked logits are -inf -> P = 0.
      float alpha = 1.f;
      bool need = false;
      if (quad_live) {
        const bool pre = j < nb_pre;
        const int key0 = (pre ? j : j - nb_pre) * KB;
        float mx = -CUDART_INF_F;
        if (!(pre && key0 + KB <= vlen)) {
#pragma unroll
          for (int c = 0; c < KB; ++c) {
            const int key = key0 + c;
            const bool vis = pre ? key < vlen : (key <= t && key < T_ && __ldg(tv + key));
            if (!vis) sv[c] = -CUDART_INF_F;
          }
        }
#pragma unroll
        for (int c = 0; c < KB; ++c) mx = fmaxf(mx, sv[c]);
        mx = row_ok ? mx * L2E : -CUDART_INF_F;
        need = mx > m_use + RESCALE_LOG2;   // false while mx == -inf
        if (need) {
          alpha = ex2_approx(m_use - mx);    // m_use == -inf -> 0
          m_use = mx;
        }
      }
      // P buffer and O are free once the previous P.V finished
      if (j >= 1) {
        mbar_wait(pv_done, (j - 1) & 1);
        tc_fence_after();
      }
      if (j >= 1 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t o[32];
          tmem_ld32_nowait(lane_base + O_COL + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st32(lane_base + O_COL + c * 32, o);
        }
        tmem_st_wait();
      }
      if (quad_live) {
        const float neg_m = !row_ok ? -CUDART_INF_F : (m_use == -CUDART_INF_F) ? 0.f : -m_use;
        float l0 = 0.f, l1 = 0.f;
#pragma unroll
        for (int c8 = 0; c8 < KB / 8; ++c8) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float p0 = ex2_approx(fmaf(sv[c8 * 8 + 2 * e], L2E, neg_m));
            const float p1 = ex2_approx(fmaf(sv[c8 * 8 + 2 * e + 1], L2E, neg_m));
            l0 += p0;
            l1 += p1;
            w[e] = pack_2<T>(p0, p1);
          }
          const int atom = c8 >> 3, cc = c8 & 7;
          *reinterpret_cast<uint4*>(prow + atom * S::ATOM + ((cc ^ sw) << 4)) =
              make_uint4(w[0], w[1], w[2], w[3]);
        }
        l = l * alpha + (l0 + l1);
      }
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    // ---------------------------------------------------------- epilogue
    mbar_wait(pv_done, (nb - 1) & 1);
    tc_fence_after();
    if (quad_live) {
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const int H = p.KVH * p.G;
      T* dst = reinterpret_cast<T*>(p.out) + ((int64_t)b * T_ + t) * (H * HD) +
               (int64_t)(kvh * p.G + g) * HD;
#pragma unroll 1
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t o[32];
        tmem_ld32_nowait(lane_base + O_COL + c * 32, o);
        tmem_ld_wait();
        if (row_ok) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              w[e] = pack_2<T>(__uint_as_float(o[q4 * 8 + 2 * e]) * inv,
                               __uint_as_float(o[q4 * 8 + 2 * e + 1]) * inv);
            d4[q4] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(S::TMEM_COLS) : "memory");
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

static int encode(CUtensorMap* map, const void* base, CUtensorMapDataType dt, int rank,
                  const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box) {
  auto enc = encoder();
  if (!enc) return fail(KRR_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, dt, rank, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(KRR_ECUDA, "attention tensor map encode failed: " + std::to_string((int)r));
  return KRR_OK;
}

template <typename T, int HD, int KB>
static int launch(const AttnParams& a, cudaStream_t s) {
  using Sm = Smem<HD, KB>;
  const CUtensorMapDataType dt = std::is_same<T, __half>::value ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                                : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const int R = a.group * a.seq_len;
  const int64_t units = (int64_t)a.n_seqs * a.kv_heads;
  const int row_tiles = (R + TM - 1) / TM;
  KRR_REQUIRE(units * R < INT32_MAX && units * row_tiles < INT32_MAX, KRR_ESHAPE,
              "attention batch too large");
  CUtensorMap mq, mp, mc;
  {
    cuuint64_t dims[2] = {(cuuint64_t)HD, (cuuint64_t)(units * R)};
    cuuint64_t str[1] = {(cuuint64_t)HD * sizeof(T)};
    cuuint32_t box[2] = {64, TM};
    int rc = encode(&mq, a.q, dt, 2, dims, str, box);
    if (rc) return rc;
  }
  const int64_t cur_page = (int64_t)a.seq_len * HD * sizeof(T);
  {
    cuuint64_t dims[3] = {(cuuint64_t)HD, (cuuint64_t)a.seq_len,
                          (cuuint64_t)(a.cur_pool_bytes / cur_page)};
    cuuint64_t str[2] = {(cuuint64_t)HD * sizeof(T), (cuuint64_t)cur_page};
    cuuint32_t box[3] = {64, (cuuint32_t)KB, 1};
    int rc = encode(&mc, a.cur_pool, dt, 3, dims, str, box);
    if (rc) return rc;
  }
  const int64_t pre_page = (int64_t)std::max(a.prefix_len, 1) * HD * sizeof(T);
  if (a.prefix_len > 0) {
    cuuint64_t dims[3] = {(cuuint64_t)HD, (cuuint64_t)a.prefix_len,
                          (cuuint64_t)(a.prefix_pool_bytes / pre_page)};
    cuuint64_t str[2] = {(cuuint64_t)HD * sizeof(T), (cuuint64_t)pre_page};
    cuuint32_t box[3] = {64, (cuuint32_t)KB, 1};
    int rc = encode(&mp, a.prefix_pool, dt, 3, dims, str, box);
    if (rc) return rc;
  } else {
    mp = mc;
  }
  Params p{a.prefix_kv, static_cast<const char*>(a.prefix_pool), pre_page, a.cur_kv,
           static_cast<const char*>(a.cur_pool), cur_page, a.prefix_valid_len, a.tok_valid,
           a.out, a.kv_heads, a.group, a.seq_len, a.prefix_len, a.layer, a.cur_layer, R,
           row_tiles};
  {
    const int rc = ensure_func_smem((const void*)attn_tc_kernel<T, HD, KB>, Sm::TOTAL, 100);
    if (rc) return rc;
  }
  attn_tc_kernel<T, HD, KB><<<(unsigned)(units * row_tiles), THREADS, Sm::TOTAL, s>>>(mq, mp, mc, p);
  return check_launch("attention_tc");
}

bool supported(int act, const AttnParams& a) {
  return (act == KRR_F16 || act == KRR_BF16) &&
         (a.head_dim == 64 || a.head_dim == 128 || a.head_dim == 256) &&
         a.cur_pool != nullptr && a.cur_pool_bytes > 0 &&
         (a.prefix_len == 0 || (a.prefix_pool != nullptr && a.prefix_pool_bytes > 0));
}

}  // namespace attn_tc

int launch_attention_tcgen05(int act_dtype, const AttnParams& p, cudaStream_t s) {
  if (!attn_tc::supported(act_dtype, p))
    return fail(KRR_EUNSUPPORTED, "tcgen05 attention needs f16/bf16, head_dim 64|128|256 and pool bases");
  constexpr int KB = 64;
  if (act_dtype == KRR_F16) {
    if (p.head_dim == 64) return attn_tc::launch<__half, 64, KB>(p, s);
    if (p.head_dim == 128) return attn_tc::launch<__half, 128, KB>(p, s);
    return attn_tc::launch<__half, 256, KB>(p, s);
  }
  if (p.head_dim == 64) return attn_tc::launch<__nv_bfloat16, 64, KB>(p, s);
  if (p.head_dim == 128) return attn_tc::launch<__nv_bfloat16, 128, KB>(p, s);
  return attn_tc::launch<__nv_bfloat16, 256, KB>(p, s);
}

bool attention_tcgen05_supported(int act_dtype, const AttnParams& p) {
  return attn_tc::supported(act_dtype, p);
}

template <typename T, int HD>
static int occupancy(int* out) {
  using namespace attn_tc;
  auto* k = attn_tc_kernel<T, HD, 64>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem<HD, 64>::TOTAL);
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, k, THREADS,
                                                                Smem<HD, 64>::TOTAL);
  if (e != cudaSuccess) return fail(KRR_ECUDA, cudaGetErrorString(e));
  return KRR_OK;
}

int attention_tcgen05_occupancy(int act_dtype, int head_dim, int* out) {
  KRR_REQUIRE(head_dim == 64 || head_dim == 128, KRR_EUNSUPPORTED, "head_dim 64|128");
  // (head_dim 256 runs one CTA per SM by design: 512 TMEM columns)
  if (act_dtype == KRR_BF16)
    return head_dim == 64 ? occupancy<__nv_bfloat16, 64>(out) : occupancy<__nv_bfloat16, 128>(out);
  return head_dim == 64 ? occupancy<__half, 64>(out) : occupancy<__half, 128>(out);
}

}  // namespace krr
