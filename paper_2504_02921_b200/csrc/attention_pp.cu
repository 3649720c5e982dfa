// Persistent ping-pong tensor-core attention for sm_100a (tcgen05 / TMEM / TMA).
//
// Same semantics as attention.cu / attention_tc.cu (model.py:349-394,
// _exp_rows :406-436).  Differences from the one-tile kernel:
//
//  * work item = (unit, pair of 128-row tiles): both tiles (A, B) of a unit's
//    GQA-packed rows share every K/V block, so each block is fetched from HBM
//    and staged in smem ONCE for up to 256 query rows (C3: G*Q = 192 rows = one
//    item);
//  * one persistent CTA per SM walks the items with a static stride, so the
//    barrier init / TMEM allocation happens once and the K/V rings run ahead
//    across item boundaries;
//  * two softmax warpgroups (A: warps 2-5, B: warps 6-9), each owning one tile's
//    TMEM lanes, alternate with the single MMA thread: while WG A turns S_A into
//    P_A, the tensor core computes S_B or P_B.V, and vice versa.
//
// TMEM (512 columns): tile A  S[2] at 0/KB, O at 2KB;  tile B at +256.
// SMEM (224 KB): Q_A|Q_B 64 KB, K ring 3x16 KB, V ring 3x16 KB, P[tile][2] 64 KB.
// P is double-buffered per tile so the softmax of block j+1 need not wait for
// P.V of block j (only a rare O rescale does).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math_constants.h>
#include <mutex>
#include "launchers.h"
#include "tc_ptx.cuh"

namespace krr {
namespace attn_pp {
using namespace tc;
#ifdef KRR_PP_TRACE
// timing trace of CTA 0 (experiments only): trace[role*8+event][g] = clock64()
__device__ unsigned long long g_pp_trace[16 * 8 * 64];
#define TR(role, ev, gidx)                                                        \
  do {                                                                            \
    if (blockIdx.x == 0 && (gidx) < 64 && (threadIdx.x & 31) == 0)                \
      g_pp_trace[((role) * 8 + (ev)) * 64 + (gidx)] = clock64();                  \
  } while (0)
#else
#define TR(role, ev, gidx) do {} while (0)
#endif
#ifndef KRR_PP_SLEEP
#define mbar_wait mbar_wait_fast
#endif

constexpr int TM = 128;
constexpr int KB = 64;
constexpr int NST = 3;          // K and V ring depth
constexpr int THREADS = 384;    // w0 Q, w1 MMA, w2-5 softmax A, w6-9 softmax B, w10 K, w11 V
// Lazy O rescale: the running max used for P is raised only when a block's max
// exceeds it by 2^15, so P = 2^(s*log2e - m) <= 32768 (< f16 max 65504) and O/l
// stay far from f32 limits; the final O/l is exact for any stale max.
#ifdef KRR_PP_NORESCALE   // timing experiments only (wrong results with large logits)
constexpr float RESCALE_LOG2 = 1e30f;
#else
constexpr float RESCALE_LOG2 = 15.0f;
#endif

struct Params {
  void* const* prefix_kv;
  const char* prefix_base;
  int64_t prefix_page_bytes;
  void* const* cur_kv;
  const char* cur_base;
  int64_t cur_page_bytes;
  const int32_t* prefix_valid_len;
  const uint8_t* tok_valid;
  void* out;
  int KVH, G, T, P, layer, cur_layer, R, pairs, items;
};

template <int HD>
struct Smem {
  static constexpr int ATOM = TM * 128;                  // one 128-row swizzle column
  static constexpr int Q_TILE = (HD / 64) * ATOM;
  static constexpr int KV_BYTES = (HD / 64) * KB * 128;  // one K or V block
  static constexpr int P_TILE = (KB / 64) * ATOM;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + 2 * Q_TILE;
  static constexpr int V_OFF = K_OFF + NST * KV_BYTES;
  static constexpr int P_OFF = V_OFF + NST * KV_BYTES;
  static constexpr int BAR_OFF = P_OFF + 4 * P_TILE;   // P[tile][2 buffers]
  static constexpr int TOTAL = BAR_OFF + 512;
  static_assert(2 * KB + HD <= 256, "TMEM budget per tile");
};

// barrier slots
enum {
  B_QFULL = 0, B_QEMPTY, B_KFULL, B_KEMPTY = B_KFULL + NST, B_VFULL = B_KEMPTY + NST,
  B_VEMPTY = B_VFULL + NST, B_SFULL = B_VEMPTY + NST /*[tile][buf]*/,
  B_SEMPTY = B_SFULL + 4, B_PFULL = B_SEMPTY + 4 /*[tile][buf]*/, B_PVDONE = B_PFULL + 4,
  B_OEMPTY = B_PVDONE + 4, B_COUNT = B_OEMPTY + 2
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

// Geometry of one work item, identical in every role.
struct Item {
  int unit, b, kvh, row0, nb_pre, nb, vlen, t_max;
};
__device__ __forceinline__ Item item_of(const Params& p, int it) {
  Item x;
  x.unit = it / p.pairs;
  const int pair = it - x.unit * p.pairs;
  x.b = x.unit / p.KVH;
  x.kvh = x.unit - x.b * p.KVH;
  x.row0 = pair * 2 * TM;                      // tile A rows; tile B = row0 + TM
  const int last_row = min(x.row0 + 2 * TM, p.R) - 1;
  x.t_max = (last_row / p.T != x.row0 / p.T) ? p.T - 1 : last_row % p.T;
  x.vlen = p.P ? min(p.prefix_valid_len[x.b], p.P) : 0;
  x.nb_pre = (x.vlen + KB - 1) / KB;
  x.nb = x.nb_pre + (x.t_max + 1 + KB - 1) / KB;
  return x;
}

template <typename T, int HD>
__global__ void __launch_bounds__(THREADS, 1)
    attn_pp_kernel(const __grid_constant__ CUtensorMap tmQ,
                   const __grid_constant__ CUtensorMap tmPre,
                   const __grid_constant__ CUtensorMap tmCur, const Params p) {
  using S = Smem<HD>;
  extern __shared__ uint8_t smem[];
  uint8_t* sQ = smem + S::Q_OFF;
  uint8_t* sK = smem + S::K_OFF;
  uint8_t* sV = smem + S::V_OFF;
  uint8_t* sP = smem + S::P_OFF;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + B_COUNT);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    if ((smem_u32(smem) & 1023) != 0) __trap();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmPre)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmCur)) : "memory");
    mbar_init(&bar[B_QFULL], 1);
    mbar_init(&bar[B_QEMPTY], 1);
    for (int s = 0; s < NST; ++s) {
      mbar_init(&bar[B_KFULL + s], 1); mbar_init(&bar[B_KEMPTY + s], 1);
      mbar_init(&bar[B_VFULL + s], 1); mbar_init(&bar[B_VEMPTY + s], 1);
    }
    for (int i = 0; i < 4; ++i) { mbar_init(&bar[B_SFULL + i], 1); mbar_init(&bar[B_SEMPTY + i], 4); }
    for (int i = 0; i < 4; ++i) { mbar_init(&bar[B_PFULL + i], 4); mbar_init(&bar[B_PVDONE + i], 1); }
    for (int x = 0; x < 2; ++x) mbar_init(&bar[B_OEMPTY + x], 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------- producers
    // warp 0: Q tiles (waits for the previous item's last S MMA); warps 10/11:
    // K / V rings.  Separate warps (not lanes of one warp: a sleeping lane
    // would stall its diverged siblings) so K/V prefetch runs ahead across
    // item boundaries while Q waits.
    if (lane == 0) {
      int n = 0;
      for (int it = blockIdx.x; it < p.items; it += gridDim.x, ++n) {
        const Item x = item_of(p, it);
        mbar_wait(&bar[B_QEMPTY], (n & 1) ^ 1);
        mbar_expect_tx(&bar[B_QFULL], 2 * S::Q_TILE);
#pragma unroll
        for (int tile = 0; tile < 2; ++tile)
#pragma unroll
          for (int a = 0; a < HD / 64; ++a)
            tma_load<1>(sQ + tile * S::Q_TILE + a * S::ATOM, &tmQ, smem_u32(&bar[B_QFULL]),
                        a * 64, x.unit * p.R + x.row0 + tile * TM);
      }
    }
  } else if (warp >= 10) {
    if (lane == 0) {
      const bool is_k = warp == 10;
      uint64_t* full = &bar[is_k ? B_KFULL : B_VFULL];
      uint64_t* empty = &bar[is_k ? B_KEMPTY : B_VEMPTY];
      uint8_t* ring = is_k ? sK : sV;
      int g = 0;
      for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
        const Item x = item_of(p, it);
        const int pre_page = p.P ? (int)((reinterpret_cast<const char*>(p.prefix_kv[x.b]) -
                                          p.prefix_base) / p.prefix_page_bytes) +
                                       (p.layer * 2) * p.KVH + x.kvh
                                 : 0;
        const int cur_page = (int)((reinterpret_cast<const char*>(p.cur_kv[x.b]) - p.cur_base) /
                                   p.cur_page_bytes) + (p.cur_layer * 2) * p.KVH + x.kvh;
        const int vofs = is_k ? 0 : p.KVH;
        for (int j = 0; j < x.nb; ++j, ++g) {
          const int s = g % NST;
          mbar_wait(&empty[s], ((g / NST) & 1) ^ 1);
          TR(is_k ? 0 : 1, 0, g);
          mbar_expect_tx(&full[s], S::KV_BYTES);
          const bool pre = j < x.nb_pre;
          const CUtensorMap* map = pre ? &tmPre : &tmCur;
          const int key0 = (pre ? j : j - x.nb_pre) * KB;
          const int pk = (pre ? pre_page : cur_page) + vofs;
#pragma unroll
          for (int a = 0; a < HD / 64; ++a)
            tma_load3(ring + s * S::KV_BYTES + a * (KB * 128), map, &full[s], a * 64, key0, pk);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    // The whole warp walks the schedule (waits included); one elected lane
    // issues.  Descriptors are built once and advanced by adding the 16-byte
    // granular smem offset to the start-address field.
    constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
    constexpr uint32_t idesc_s = (1u << 4) | (fmt << 7) | (fmt << 10) |
                                 ((uint32_t)(KB >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
    constexpr uint32_t idesc_o = (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 16) |
                                 ((uint32_t)(HD >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
    const uint64_t dQ = sw128_desc(smem_u32(sQ));
    const uint64_t dK = sw128_desc(smem_u32(sK));
    const uint64_t dP = sw128_desc(smem_u32(sP));
    const uint64_t dV = sw128_desc_mn(smem_u32(sV), KB * 128, 1024);
    int g = 0, n = 0;
    for (int it = blockIdx.x; it < p.items; it += gridDim.x, ++n) {
      const Item x = item_of(p, it);
      mbar_wait(&bar[B_QFULL], n & 1);
      for (int j = 0; j <= x.nb; ++j) {
        if (j < x.nb) {
          const int gs = g + j, st = gs % NST, sb = gs & 1;
          mbar_wait(&bar[B_KFULL + st], (gs / NST) & 1);
          TR(2, 0, gs);
#pragma unroll
          for (int tile = 0; tile < 2; ++tile) {
            mbar_wait(&bar[B_SEMPTY + tile * 2 + sb], ((gs >> 1) & 1) ^ 1);
            tc_fence_after();
            if (tile == 0) TR(2, 4, gs);
            if (elect_one_sync()) {
              const uint32_t d = tmem + tile * 256 + sb * KB;
#pragma unroll
              for (int k = 0; k < HD / 16; ++k) {
                const uint32_t off = (k >> 2) * S::ATOM + (k & 3) * 32;
                const uint32_t koff = st * S::KV_BYTES + (k >> 2) * (KB * 128) + (k & 3) * 32;
                mma_f16<1>(d, dQ + ((tile * S::Q_TILE + off) >> 4), dK + (koff >> 4), idesc_s,
                           k > 0);
              }
              mma_commit<1>(&bar[B_SFULL + tile * 2 + sb]);
            }
            __syncwarp();
            if (tile == 0) TR(2, 5, gs);
          }
          if (elect_one_sync()) {
            mma_commit<1>(&bar[B_KEMPTY + st]);
            if (j == x.nb - 1) mma_commit<1>(&bar[B_QEMPTY]);
          }
          __syncwarp();
          TR(2, 1, gs);
        }
        if (j >= 1) {
          const int jj = j - 1, gp = g + jj, st = gp % NST;
          mbar_wait(&bar[B_VFULL + st], (gp / NST) & 1);
          TR(2, 2, gp);
#pragma unroll
          for (int tile = 0; tile < 2; ++tile) {
            if (jj == 0) mbar_wait(&bar[B_OEMPTY + tile], (n & 1) ^ 1);
            mbar_wait(&bar[B_PFULL + tile * 2 + (gp & 1)], (gp >> 1) & 1);
            tc_fence_after();
            if (tile == 0) TR(2, 6, gp);
            if (elect_one_sync()) {
              const uint32_t d = tmem + tile * 256 + 2 * KB;
              const uint32_t pbase = (tile * 2 + (gp & 1)) * S::P_TILE;
#pragma unroll
              for (int k = 0; k < KB / 16; ++k)
                mma_f16<1>(d, dP + ((pbase + (k >> 2) * S::ATOM + (k & 3) * 32) >> 4),
                           dV + ((st * S::KV_BYTES + k * 16 * 128) >> 4), idesc_o,
                           (jj > 0) || (k > 0));
              mma_commit<1>(&bar[B_PVDONE + tile * 2 + (gp & 1)]);
            }
            __syncwarp();
            if (tile == 0) TR(2, 7, gp);
          }
          if (elect_one_sync()) mma_commit<1>(&bar[B_VEMPTY + st]);
          __syncwarp();
          TR(2, 3, gp);
        }
      }
      g += x.nb;
    }
  } else {
    // ---------------------------------------------------------- softmax WGs
    const int tile = (warp - 2) >> 2;               // 0: warps 2-5, 1: warps 6-9
    const int quad = warp & 3;
    const int lrow = quad * 32 + lane;
    const uint32_t lane_base = tmem + tile * 256 + ((uint32_t)(quad * 32) << 16);
    const uint32_t o_col = 2 * KB;
    uint64_t* s_full = &bar[B_SFULL + tile * 2];
    uint64_t* s_empty = &bar[B_SEMPTY + tile * 2];
    uint64_t* p_full = &bar[B_PFULL + tile * 2];    // [buf]
    uint64_t* pv_done = &bar[B_PVDONE + tile * 2];  // [buf]: P.V of block gs done <=> buf gs&1 free
    uint8_t* prow0 = sP + tile * 2 * S::P_TILE + lrow * 128;
    const int sw = lrow & 7;
    const float L2E = 1.4426950408889634f;
    const int T_ = p.T;
    const int H = p.KVH * p.G;
    int g = 0;
    for (int it = blockIdx.x; it < p.items; it += gridDim.x) {
      const Item x = item_of(p, it);
      const int r = x.row0 + tile * TM + lrow;
      const bool row_ok = r < p.R;
      const bool quad_live = x.row0 + tile * TM + quad * 32 < p.R;
      const int gq = r / T_, t = r - gq * T_;
      const uint8_t* tv = p.tok_valid + (int64_t)x.b * T_;
      float m_use = -CUDART_INF_F, l = 0.f;
      for (int j = 0; j < x.nb; ++j) {
        const int gs = g + j, sb = gs & 1;
        mbar_wait(&s_full[sb], (gs >> 1) & 1);
        if (quad == 2) TR(3 + tile, 0, gs);
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
        if (quad == 2) TR(3 + tile, 1, gs);

        float alpha = 1.f;
        bool need = false;
        if (quad_live) {
          const bool pre = j < x.nb_pre;
          const int key0 = (pre ? j : j - x.nb_pre) * KB;
          if (!(pre && key0 + KB <= x.vlen)) {
#pragma unroll
            for (int c = 0; c < KB; ++c) {
              const int key = key0 + c;
              const bool vis = pre ? key < x.vlen : (key <= t && key < T_ && __ldg(tv + key));
              if (!vis) sv[c] = -CUDART_INF_F;
            }
          }
          float m8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) m8[e] = fmaxf(sv[e], sv[e + 8]);
#pragma unroll
          for (int c = 16; c < KB; c += 8)
#pragma unroll
            for (int e = 0; e < 8; ++e) m8[e] = fmaxf(m8[e], sv[c + e]);
          float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                           fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
          mx = row_ok ? mx * L2E : -CUDART_INF_F;
          need = mx > m_use + RESCALE_LOG2;
          if (need) {
            alpha = ex2_approx(m_use - mx);
            m_use = mx;
          }
        }
        // P double buffer: buffer gs&1 was last read by P.V of block gs-2
        if (j >= 2) {
          mbar_wait(&pv_done[gs & 1], ((gs - 2) >> 1) & 1);
          tc_fence_after();
        }
        if (quad == 2) TR(3 + tile, 2, gs);
        const bool rescale = j >= 1 && __any_sync(0xffffffffu, need);
        if (rescale) {                         // O must be stable: P.V of block gs-1 done
          mbar_wait(&pv_done[(gs - 1) & 1], ((gs - 1) >> 1) & 1);
          tc_fence_after();
        }
        if (rescale) {
#pragma unroll 1
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t o[32];
            tmem_ld32_nowait(lane_base + o_col + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(lane_base + o_col + c * 32, o);
          }
          tmem_st_wait();
        }
        if (quad == 2) TR(3 + tile, 6, gs);
        if (quad_live) {
          const float neg_m = !row_ok ? -CUDART_INF_F : (m_use == -CUDART_INF_F) ? 0.f : -m_use;
          float l4[4] = {0.f, 0.f, 0.f, 0.f};
          uint8_t* prow = prow0 + (gs & 1) * S::P_TILE;
#pragma unroll
          for (int c8 = 0; c8 < KB / 8; ++c8) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float p0 = ex2_approx(fmaf(sv[c8 * 8 + 2 * e], L2E, neg_m));
              const float p1 = ex2_approx(fmaf(sv[c8 * 8 + 2 * e + 1], L2E, neg_m));
              l4[e] += p0 + p1;
              w[e] = pack_2<T>(p0, p1);
            }
            const int atom = c8 >> 3, cc = c8 & 7;
            *reinterpret_cast<uint4*>(prow + atom * S::ATOM + ((cc ^ sw) << 4)) =
                make_uint4(w[0], w[1], w[2], w[3]);
          }
          l = l * alpha + ((l4[0] + l4[1]) + (l4[2] + l4[3]));
        }
        if (quad == 2) TR(3 + tile, 7, gs);
        fence_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[gs & 1]);
        if (quad == 2) TR(3 + tile, 3, gs);
      }
      // ---------------------------------------------------------- epilogue
      mbar_wait(&pv_done[(g + x.nb - 1) & 1], ((g + x.nb - 1) >> 1) & 1);
      if (quad == 2) TR(3 + tile, 4, g + x.nb - 1);
      tc_fence_after();
      if (quad_live) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        T* dst = reinterpret_cast<T*>(p.out) + ((int64_t)x.b * T_ + t) * (H * HD) +
                 (int64_t)(x.kvh * p.G + gq) * HD;
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t o[32];
          tmem_ld32_nowait(lane_base + o_col + c * 32, o);
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
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar[B_OEMPTY + tile]);
      if (quad == 2) TR(3 + tile, 5, g + x.nb - 1);
      g += x.nb;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
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

template <typename T, int HD>
static int launch(const AttnParams& a, cudaStream_t s) {
  using Sm = Smem<HD>;
  const CUtensorMapDataType dt = std::is_same<T, __half>::value ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                                : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const int R = a.group * a.seq_len;
  const int64_t units = (int64_t)a.n_seqs * a.kv_heads;
  const int pairs = (R + 2 * TM - 1) / (2 * TM);
  KRR_REQUIRE(units * R < INT32_MAX && units * pairs < INT32_MAX, KRR_ESHAPE,
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
  const int items = (int)(units * pairs);
  Params p{a.prefix_kv, static_cast<const char*>(a.prefix_pool), pre_page, a.cur_kv,
           static_cast<const char*>(a.cur_pool), cur_page, a.prefix_valid_len, a.tok_valid,
           a.out, a.kv_heads, a.group, a.seq_len, a.prefix_len, a.layer, a.cur_layer, R,
           pairs, items};
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_pp_kernel<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Sm::TOTAL);
    attr = true;
  }
  const int grid = std::min(items, device_sm_count());
  attn_pp_kernel<T, HD><<<grid, THREADS, Sm::TOTAL, s>>>(mq, mp, mc, p);
  return check_launch("attention_pp");
}

}  // namespace attn_pp

#ifdef KRR_PP_TRACE
extern "C" int krr_pp_trace_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, attn_pp::g_pp_trace, sizeof(attn_pp::g_pp_trace)) == cudaSuccess ? 0 : 3;
}
#endif

int launch_attention_pingpong(int act_dtype, const AttnParams& p, cudaStream_t s) {
  if (!attention_tcgen05_supported(act_dtype, p) || p.head_dim > 128)
    return fail(KRR_EUNSUPPORTED, "tcgen05 attention needs f16/bf16, head_dim 64|128 and pool bases");
  if (act_dtype == KRR_F16)
    return p.head_dim == 64 ? attn_pp::launch<__half, 64>(p, s) : attn_pp::launch<__half, 128>(p, s);
  return p.head_dim == 64 ? attn_pp::launch<__nv_bfloat16, 64>(p, s)
                          : attn_pp::launch<__nv_bfloat16, 128>(p, s);
}

}  // namespace krr
