// Tensor-core attention with 128-key blocks and one S/P buffer per tile (sm_100a).
//
// Same semantics as attention.cu / attention_fa.cu (model.py:349-394, _exp_rows
// :406-436).  attention_fa.cu works on 64-key blocks with two S buffers per
// tile; its CTA timeline (profiles/r01_attn_fa_trace.txt) and MMA-work
// halving experiments show the time per block is mostly a fixed handoff chain
// (MMA-warp barrier waits, commits, softmax wake-ups), not tensor work.  This
// variant halves the number of blocks per key:
//
//  * KB = 128 keys per block: S = Q.K^T runs as N=128 MMAs (the 128x16 Q slice
//    is re-read from smem once per 128 keys instead of per 64);
//  * TMEM per tile: S/P 128 columns + O (HD columns); two tiles = 512 columns,
//    so S is single-buffered per tile and the two tiles ping-pong: the MMA
//    warp issues PV_X(j) then S_X(j+1) into the same buffer (in-order tensor
//    pipe: P_X(j) is read before S_X(j+1) lands) while the other tile's
//    softmax runs;
//  * S_X(j) completing implies PV_X(j-1) completed (issued earlier, in order),
//    so the lazy O rescale needs no extra barrier;
//  * the softmax makes two passes over the 128 columns (max, then exp + P
//    store), 64 / 32 columns at a time, to stay within the register budget of
//    10 warps.
//
// Work item = (unit, pair of 128-row tiles), K/V rings of 2 blocks.
// SMEM (HD=128): Q_A|Q_B 64 KB, K ring 2 x 32 KB, V ring 2 x 32 KB = 192 KB.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math_constants.h>
#include <mutex>
#include "launchers.h"
#include "tc_ptx.cuh"

namespace krr {
namespace attn_fa2 {
using namespace tc;
#define mbar_wait mbar_wait_fast   // latency-critical handoffs: no suspend hint

constexpr int TM = 128;
constexpr int KB = 128;
constexpr int NK = 2, NV = 2;   // K / V ring depth (blocks)
constexpr int THREADS = 320;    // w0 producers (lanes 0 Q, 1 K, 2 V), w1 MMA, w2-5 / w6-9 softmax
constexpr float RESCALE_LOG2 = 15.0f;   // P <= 2^15 < f16 max

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
  static constexpr int ATOM_Q = TM * 128;                // one 64-wide swizzle column of Q
  static constexpr int ATOM_KV = KB * 128;               // one 64-wide swizzle column of K/V
  static constexpr int Q_TILE = (HD / 64) * ATOM_Q;
  static constexpr int KV_BYTES = (HD / 64) * ATOM_KV;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + 2 * Q_TILE;
  static constexpr int V_OFF = K_OFF + NK * KV_BYTES;
  static constexpr int BAR_OFF = V_OFF + NV * KV_BYTES;
  static constexpr int TOTAL = BAR_OFF + 512;
  static_assert(KB + HD <= 256, "TMEM budget per tile");
};

enum {
  B_QFULL = 0, B_QEMPTY, B_KFULL, B_KEMPTY = B_KFULL + NK, B_VFULL = B_KEMPTY + NK,
  B_VEMPTY = B_VFULL + NV, B_SFULL = B_VEMPTY + NV /*[tile]*/, B_PFULL = B_SFULL + 2 /*[tile]*/,
  B_ODONE = B_PFULL + 2, B_OEMPTY = B_ODONE + 2, B_COUNT = B_OEMPTY + 2
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

// O += P.V with P (A operand) in TMEM, V (B operand) from smem.
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// tcgen05.st 32 lanes x 16 columns
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),
        "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),
        "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

struct Item {
  int unit, b, kvh, row0, nb_pre, nb, vlen, t_max;
};
__device__ __forceinline__ Item item_of(const Params& p, int it) {
  Item x;
  x.unit = it / p.pairs;
  const int pair = it - x.unit * p.pairs;
  x.b = x.unit / p.KVH;
  x.kvh = x.unit - x.b * p.KVH;
  x.row0 = pair * 2 * TM;
  const int last_row = min(x.row0 + 2 * TM, p.R) - 1;
  x.t_max = (last_row / p.T != x.row0 / p.T) ? p.T - 1 : last_row % p.T;
  x.vlen = p.P ? min(p.prefix_valid_len[x.b], p.P) : 0;
  x.nb_pre = (x.vlen + KB - 1) / KB;
  x.nb = x.nb_pre + (x.t_max + 1 + KB - 1) / KB;
  return x;
}

template <typename T, int HD>
__global__ void __launch_bounds__(THREADS, 1)
    attn_fa2_kernel(const __grid_constant__ CUtensorMap tmQ,
                    const __grid_constant__ CUtensorMap tmPre,
                    const __grid_constant__ CUtensorMap tmCur, const Params p) {
  using S = Smem<HD>;
  extern __shared__ uint8_t smem[];
  uint8_t* sQ = smem + S::Q_OFF;
  uint8_t* sK = smem + S::K_OFF;
  uint8_t* sV = smem + S::V_OFF;
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
    for (int s = 0; s < NK; ++s) { mbar_init(&bar[B_KFULL + s], 1); mbar_init(&bar[B_KEMPTY + s], 1); }
    for (int s = 0; s < NV; ++s) { mbar_init(&bar[B_VFULL + s], 1); mbar_init(&bar[B_VEMPTY + s], 1); }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&bar[B_SFULL + x], 1);
      mbar_init(&bar[B_PFULL + x], 4);
      mbar_init(&bar[B_ODONE + x], 1);
      mbar_init(&bar[B_OEMPTY + x], 4);
    }
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
    if (lane == 0) {                                   // Q tiles, per item
      int n = 0;
      for (int it = blockIdx.x; it < p.items; it += gridDim.x, ++n) {
        const Item x = item_of(p, it);
        mbar_wait(&bar[B_QEMPTY], (n & 1) ^ 1);
        mbar_expect_tx(&bar[B_QFULL], 2 * S::Q_TILE);
#pragma unroll
        for (int tile = 0; tile < 2; ++tile)
#pragma unroll
          for (int a = 0; a < HD / 64; ++a)
            tma_load<1>(sQ + tile * S::Q_TILE + a * S::ATOM_Q, &tmQ, smem_u32(&bar[B_QFULL]),
                        a * 64, x.unit * p.R + x.row0 + tile * TM);
      }
    } else if (lane < 3) {                             // K ring (lane 1), V ring (lane 2)
      const bool is_k = lane == 1;
      const int nst = is_k ? NK : NV;
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
          const int s = g % nst;
          mbar_wait(&empty[s], ((g / nst) & 1) ^ 1);
          mbar_expect_tx(&full[s], S::KV_BYTES);
          const bool pre = j < x.nb_pre;
          const CUtensorMap* map = pre ? &tmPre : &tmCur;
          const int key0 = (pre ? j : j - x.nb_pre) * KB;
          const int pk = (pre ? pre_page : cur_page) + vofs;
#pragma unroll
          for (int a = 0; a < HD / 64; ++a)
            tma_load3(ring + s * S::KV_BYTES + a * S::ATOM_KV, map, &full[s], a * 64, key0, pk);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    constexpr uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
    constexpr uint32_t idesc_s = (1u << 4) | (fmt << 7) | (fmt << 10) |
                                 ((uint32_t)(KB >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
    constexpr uint32_t idesc_o = (1u << 4) | (fmt << 7) | (fmt << 10) | (1u << 16) |
                                 ((uint32_t)(HD >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
    const uint64_t dQ = sw128_desc(smem_u32(sQ));
    const uint64_t dK = sw128_desc(smem_u32(sK));
    const uint64_t dV = sw128_desc_mn(smem_u32(sV), S::ATOM_KV, 1024);
    int g = 0, n = 0;
    // S_tile = Q_tile . K(gs)^T into the tile's S/P columns
    auto issue_s = [&](int tile, int gs) {
      const int st = gs % NK;
      if (elect_one_sync()) {
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t qoff = tile * S::Q_TILE + (k >> 2) * S::ATOM_Q + (k & 3) * 32;
          const uint32_t koff = st * S::KV_BYTES + (k >> 2) * S::ATOM_KV + (k & 3) * 32;
          mma_f16<1>(tmem + tile * 256, dQ + (qoff >> 4), dK + (koff >> 4), idesc_s, k > 0);
        }
        mma_commit<1>(&bar[B_SFULL + tile]);
      }
      __syncwarp();
    };
    // O_tile += P_tile . V(gs), P (16-bit) in the first KB/2 columns of S
    auto issue_pv = [&](int tile, int gs, bool acc) {
      const int sv = gs % NV;
      if (elect_one_sync()) {
#pragma unroll
        for (int k = 0; k < KB / 16; ++k)
          mma_ts(tmem + tile * 256 + KB, tmem + tile * 256 + k * 8,
                 dV + ((sv * S::KV_BYTES + k * 16 * 128) >> 4), idesc_o, acc || k > 0);
      }
      __syncwarp();
    };
    for (int it = blockIdx.x; it < p.items; it += gridDim.x, ++n) {
      const Item x = item_of(p, it);
      mbar_wait(&bar[B_QFULL], n & 1);
      mbar_wait(&bar[B_KFULL + g % NK], (g / NK) & 1);
      tc_fence_after();
      issue_s(0, g);
      issue_s(1, g);
      if (elect_one_sync()) {
        mma_commit<1>(&bar[B_KEMPTY + g % NK]);
        if (x.nb == 1) mma_commit<1>(&bar[B_QEMPTY]);
      }
      __syncwarp();
      for (int j = 0; j < x.nb; ++j) {
        const int gs = g + j;
        const bool next = j + 1 < x.nb;
        mbar_wait(&bar[B_VFULL + gs % NV], (gs / NV) & 1);
        if (next) mbar_wait(&bar[B_KFULL + (gs + 1) % NK], ((gs + 1) / NK) & 1);
#pragma unroll
        for (int tile = 0; tile < 2; ++tile) {
          if (j == 0) mbar_wait(&bar[B_OEMPTY + tile], (n & 1) ^ 1);
          mbar_wait(&bar[B_PFULL + tile], gs & 1);
          tc_fence_after();
          issue_pv(tile, gs, j > 0);
          if (next) issue_s(tile, gs + 1);    // in-order pipe: PV(gs) reads P before S(gs+1) lands
          else if (elect_one_sync()) mma_commit<1>(&bar[B_ODONE + tile]);
          __syncwarp();
        }
        if (elect_one_sync()) {
          mma_commit<1>(&bar[B_VEMPTY + gs % NV]);
          if (next) {
            mma_commit<1>(&bar[B_KEMPTY + (gs + 1) % NK]);
            if (j + 1 == x.nb - 1) mma_commit<1>(&bar[B_QEMPTY]);
          }
        }
        __syncwarp();
      }
      g += x.nb;
    }
  } else {
    // ---------------------------------------------------------- softmax WGs
    const int tile = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int lrow = quad * 32 + lane;
    const uint32_t lane_base = tmem + tile * 256 + ((uint32_t)(quad * 32) << 16);
    const uint32_t o_col = KB;
    const float L2E = 1.4426950408889634f;
    const int T_ = p.T;
    const int H = p.KVH * p.G;
    int g = 0, n = 0;
    for (int it = blockIdx.x; it < p.items; it += gridDim.x, ++n) {
      const Item x = item_of(p, it);
      const int r = x.row0 + tile * TM + lrow;
      const bool row_ok = r < p.R;
      const bool quad_live = x.row0 + tile * TM + quad * 32 < p.R;
      const int gq = r / T_, t = r - gq * T_;
      const uint8_t* tv = p.tok_valid + (int64_t)x.b * T_;
      float m_use = -CUDART_INF_F, l = 0.f;
      for (int j = 0; j < x.nb; ++j) {
        const int gs = g + j;
        const bool pre = j < x.nb_pre;
        const int key0 = (pre ? j : j - x.nb_pre) * KB;
        // visible keys of this block as a 128-bit mask (two words)
        uint64_t msk[2] = {~0ull, ~0ull};
        if (!pre) {
          uint32_t w[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int k = key0 + q * 32 + lane;
            w[q] = __ballot_sync(0xffffffffu, k < T_ && __ldg(tv + k));
          }
          msk[0] = ((uint64_t)w[1] << 32) | w[0];
          msk[1] = ((uint64_t)w[3] << 32) | w[2];
          const int rel = t - key0;                     // keys key0+c visible iff c <= rel
          msk[0] &= rel >= 63 ? ~0ull : (rel < 0 ? 0ull : ((2ull << rel) - 1));
          msk[1] &= rel >= 127 ? ~0ull : (rel < 64 ? 0ull : ((2ull << (rel - 64)) - 1));
        } else if (key0 + KB > x.vlen) {
          const int rem = x.vlen - key0;                // 1..127 valid keys
          msk[0] = rem >= 64 ? ~0ull : ((1ull << rem) - 1);
          msk[1] = rem <= 64 ? 0ull : ((1ull << (rem - 64)) - 1);
        }
        mbar_wait(&bar[B_SFULL + tile], gs & 1);
        tc_fence_after();
        bool need = false;
        float alpha = 1.f;
        if (quad_live) {
          // pass 1: row max over the visible keys, 64 columns per round trip
          float m8[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) m8[e] = -CUDART_INF_F;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t raw[2][32];
            tmem_ld32_nowait(lane_base + h * 64, raw[0]);
            tmem_ld32_nowait(lane_base + h * 64 + 32, raw[1]);
            tmem_ld_wait();
            const uint64_t mk = msk[h];
#pragma unroll
            for (int c = 0; c < 64; ++c) {
              const float v = ((mk >> c) & 1ull) ? __uint_as_float(raw[c >> 5][c & 31])
                                                 : -CUDART_INF_F;
              m8[c & 7] = fmaxf(m8[c & 7], v);
            }
          }
          float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                           fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
          mx = row_ok ? mx * L2E : -CUDART_INF_F;
          need = mx > m_use + RESCALE_LOG2;
          if (need) {
            alpha = ex2_approx(m_use - mx);
            m_use = mx;
          }
        }
        // lazy O rescale: S(gs) is complete, so is P.V(gs-1) (issued before it)
        if (quad_live && j >= 1 && __any_sync(0xffffffffu, need)) {
#pragma unroll 1
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t o[32];
            tmem_ld32_nowait(lane_base + o_col + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st32(lane_base + o_col + c * 32, o);
          }
        }
        if (quad_live) {
          // pass 2: P = exp2(s*log2e - m) over 32-column chunks, stored as 16-bit
          // pairs over the S columns already consumed (chunk c -> columns 16c..)
          const float neg_m = !row_ok ? -CUDART_INF_F : (m_use == -CUDART_INF_F) ? 0.f : -m_use;
          float l4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int c = 0; c < KB / 32; ++c) {
            uint32_t raw[32];
            tmem_ld32_nowait(lane_base + c * 32, raw);
            tmem_ld_wait();
            const uint32_t mk = (uint32_t)(msk[c >> 1] >> ((c & 1) * 32));
            uint32_t w[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float s0 = ((mk >> (2 * i)) & 1u) ? __uint_as_float(raw[2 * i]) : -CUDART_INF_F;
              const float s1 = ((mk >> (2 * i + 1)) & 1u) ? __uint_as_float(raw[2 * i + 1])
                                                          : -CUDART_INF_F;
              const float p0 = ex2_approx(fmaf(s0, L2E, neg_m));
              const float p1 = ex2_approx(fmaf(s1, L2E, neg_m));
              l4[i & 3] += p0 + p1;
              w[i] = pack_2<T>(p0, p1);
            }
            tmem_st16(lane_base + c * 16, w);
          }
          l = l * alpha + ((l4[0] + l4[1]) + (l4[2] + l4[3]));
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar[B_PFULL + tile]);
      }
      // ---------------------------------------------------------- epilogue
      mbar_wait(&bar[B_ODONE + tile], n & 1);
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
  if (r != CUDA_SUCCESS) return fail(KRR_ECUDA, "tensor map encode failed: " + std::to_string((int)r));
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
    cudaFuncSetAttribute(attn_fa2_kernel<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Sm::TOTAL);
    attr = true;
  }
  const int grid = std::min(items, device_sm_count());
  attn_fa2_kernel<T, HD><<<grid, THREADS, Sm::TOTAL, s>>>(mq, mp, mc, p);
  return check_launch("attention_fa2");
}

}  // namespace attn_fa2

int launch_attention_fa2(int act_dtype, const AttnParams& p, cudaStream_t s) {
  if (!attention_tcgen05_supported(act_dtype, p) || p.head_dim > 128)
    return fail(KRR_EUNSUPPORTED, "128-key attention needs f16/bf16, head_dim 64|128 and pool bases");
  if (act_dtype == KRR_F16)
    return p.head_dim == 64 ? attn_fa2::launch<__half, 64>(p, s) : attn_fa2::launch<__half, 128>(p, s);
  return p.head_dim == 64 ? attn_fa2::launch<__nv_bfloat16, 64>(p, s)
                          : attn_fa2::launch<__nv_bfloat16, 128>(p, s);
}

}  // namespace krr
