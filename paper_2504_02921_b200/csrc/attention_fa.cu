// Persistent ping-pong tensor-core attention with P kept in TMEM (sm_100a).
//
// Same semantics as attention.cu (model.py:349-394, _exp_rows :406-436).
// Relative to round 1's smem-P ping-pong kernel (removed) it keeps P out of
// shared memory (no MMA operand reads of P, no softmax P stores there):
//
//  * P (16-bit) is written by the softmax warps straight back into the TMEM
//    columns that held S (tcgen05.st) and consumed as the TMEM A operand of
//    O += P.V (tcgen05.mma ... [a_tmem]) -- no smem round trip;
//  * per tile two S/P buffers of 64 keys and one O (2 tiles x (2*64 + HD)
//    columns = 512 for HD=128; three S/P buffers for the single head_dim-256
//    tile).  S runs NSB = 2 (3) blocks ahead of the softmax: the
//    issue order  PV_X(j), S_X(j+NSB)  relies on the tensor pipe executing
//    tcgen05.mma in order, so S_X(j+NSB) overwrites P_X(j) (same buffer) only
//    after PV_X(j) has read it;
//  * the rare lazy O rescale waits for the previous P.V (per-buffer barrier);
//  * the suffix-block mask (tok_valid, causal) comes from a 64-bit ballot mask,
//    not per-key global loads.
//
// Work item = 256 GQA-packed query rows (two 128-row tiles) of ONE document
// and kv head (head_dim 256, the Gemma shape: 128 rows, one tile -- its O
// accumulator needs 256 TMEM columns, so a tile's S buffers + O are 384 of the
// 512; the single tile still overlaps softmax(j) with S(j+1) and P.V(j-1)).  Sequences that share a prefix document and sit next to each
// other in the batch form a group whose rows are concatenated (each sequence
// padded to Rp = R rounded up to 64 rows), so the document's K/V is streamed
// once per 256 rows of the whole group -- the cross-query KV reuse of one
// cached document by every query that ranks it -- and a 192-row sequence no
// longer pads its own 256-row item.  Q lands by 64-row TMA boxes (one
// sequence each); the suffix keys of every sequence the item spans follow the
// prefix blocks, masked to that sequence's rows.  krr_forward builds the item
// table once per call (attn_group_items_kernel); without a table every
// sequence is its own group.
// SMEM: Q_A|Q_B 64 KB, K ring 4 x 16 KB, V ring 4 x 16 KB = 192 KB (head_dim
// 256: Q 64 KB, K ring 2 x 32 KB, V ring 3 x 32 KB = 224 KB).
//
// Quantised prefix pages (QB = 8 | 4: HRKV INT8/INT4 codes, codec.py:58-115,
// per-(kv_head, channel) f32 scales) are dequantised inside the kernel: the
// producer lands each 64-key block of codes by TMA into a small code ring
// (2 x 8 KB per K/V at INT8), and two converter warps (w10 K, w11 V) expand
// it into the same 128B-swizzled 16-bit K/V ring slots the MMAs read,
// f16(code * scale) exactly as krr_dequant_pages rounds it -- so the fused
// path is bit-identical to "dequantise the page into HBM, then attend" while
// only the codes cross HBM (2x / 4x fewer bytes) and no expand pass runs.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math_constants.h>
#include <mutex>
#include "launchers.h"
#include "tc_ptx.cuh"

namespace krr {
namespace attn_fa {
using namespace tc;
#define mbar_wait mbar_wait_fast   // latency-critical handoffs: no suspend hint
#ifdef KRR_PP_TRACE
__device__ unsigned long long g_fa_trace[16 * 8 * 64];
#define TR(role, ev, gidx)                                                        \
  do {                                                                            \
    if (blockIdx.x == 0 && (gidx) < 64 && (threadIdx.x & 31) == 0)                \
      g_fa_trace[((role) * 8 + (ev)) * 64 + (gidx)] = clock64();                  \
  } while (0)
#else
#define TR(role, ev, gidx) do {} while (0)
#endif

constexpr int TM = 128;
constexpr int KB = 64;
constexpr int NK = 4, NV = 4;   // barrier slots per K / V ring (ring depth <= 4)
constexpr int NC = 2;           // code ring depth per K / V (quantised prefix)
// 128-row tiles per work item: two (ping-pong) up to head_dim 128, one at 256
template <int HD> constexpr int tiles_of() { return HD == 256 ? 1 : 2; }
// S/P buffers per tile: two with two tiles (2 x (2*64 + 128) = 512 TMEM
// columns); the single head_dim-256 tile has room for three (3*64 + 256), so S
// runs three blocks ahead and softmax(j+1) never waits behind P.V(j-1)
template <int HD> constexpr int nsb_of() { return HD == 256 ? 3 : 2; }
// K / V ring depths (head_dim 256: 32 KB per block, 2 + 2; quantised
// prefixes: 3 + 3 next to the code rings) -- whatever leaves room for the
// output staging buffers
template <int HD, int QB> constexpr int rk_of() { return HD == 256 ? 2 : QB < 16 ? 3 : NK; }
template <int HD, int QB> constexpr int rv_of() { return HD == 256 ? 2 : QB < 16 ? 3 : NV; }
// epilogue staging per softmax warp: 32 rows x 32 columns of 16-bit output,
// rows padded to 80 B (conflict-free transpose)
constexpr int O_PITCH = 80;
constexpr int O_STG = 32 * O_PITCH;
// w0 producers (lanes 0 Q, 1 K, 2 V), w1 MMA, w2-5 (/ w6-9) softmax per tile,
// + two converter warps for quantised prefix pages
template <int HD, int QB> constexpr int threads_of() {
  return 64 + 128 * tiles_of<HD>() + (QB == 16 ? 0 : 64);
}
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
  const float* scales;   // quantised prefix: [page][HD] f32 (page as in the code pool)
  const int4* items;     // grouped items {b0, ng, row0, kvh}, or null (one group per seq)
  const int* n_items;    // device count of items[]
  int KVH, G, T, P, layer, cur_layer, R, Rp, chunks, items_implicit;
};

template <int HD, int QB = 16>
struct Smem {
  static constexpr int NT = tiles_of<HD>();
  static constexpr int ATOM_Q = TM * 128;                // one 128-row swizzle column of Q
  static constexpr int ATOM_KV = KB * 128;               // one 128-key swizzle column of K/V
  static constexpr int Q_TILE = (HD / 64) * ATOM_Q;
  static constexpr int KV_BYTES = (HD / 64) * ATOM_KV;
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + NT * Q_TILE;
  static constexpr int V_OFF = K_OFF + rk_of<HD, QB>() * KV_BYTES;
  static constexpr int CODE_ROW = HD * QB / 8;           // code bytes per key (QB < 16)
  static constexpr int CODE_BLK = KB * CODE_ROW;
  static constexpr int C_OFF = V_OFF + rv_of<HD, QB>() * KV_BYTES;    // code rings [K|V][NC]
  static constexpr int STG_OFF = C_OFF + (QB < 16 ? 2 * NC * CODE_BLK : 0);
  static constexpr int BAR_OFF = STG_OFF + 4 * NT * O_STG;
  static constexpr int TOTAL = BAR_OFF + 512;
  // per tile: two S/P buffers of KB columns + O (HD columns), tiles 256 apart
  static constexpr int TILE_COLS = NT == 2 ? 256 : 512;
  static_assert(nsb_of<HD>() * KB + HD <= TILE_COLS && NT * TILE_COLS <= 512 &&
                NT * nsb_of<HD>() <= 4, "TMEM / barrier budget");
  static_assert(TOTAL <= 232448, "shared memory budget");
  static_assert(QB == 16 || HD <= 128, "quantised prefix pages: head_dim 64|128");
};

enum {
  B_QFULL = 0, B_QEMPTY, B_KFULL, B_KEMPTY = B_KFULL + NK, B_VFULL = B_KEMPTY + NK,
  B_VEMPTY = B_VFULL + NV, B_SFULL = B_VEMPTY + NV /*[tile][buf]*/, B_PFULL = B_SFULL + 4,
  B_PVDONE = B_PFULL + 4 /*[tile][buf]*/, B_ODONE = B_PVDONE + 4, B_OEMPTY = B_ODONE + 2,
  B_CFULL = B_OEMPTY + 2 /*[K|V][NC]*/, B_CEMPTY = B_CFULL + 2 * NC, B_COUNT = B_CEMPTY + 2 * NC
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

constexpr int MAX_SPAN = 2 * TM / 64;   // sequences one item can span (Rp >= 64), NT = 2

struct Item {
  int b0, ng, row0, kvh;       // group's first sequence and size; first group row; kv head
  int s_lo, n_span;            // sequences (relative to b0) the item's rows cover
  int nbc[MAX_SPAN];           // suffix blocks needed per covered sequence
  int vlen, nb_pre, nb;
};
__device__ __forceinline__ int item_count(const Params& p) {
  return p.items ? __ldg(p.n_items) : p.items_implicit;
}
template <int NT>
__device__ __forceinline__ Item item_of(const Params& p, int it) {
  constexpr int ROWS = NT * TM;                  // query rows per item
  Item x;
  if (p.items) {
    const int4 e = __ldg(p.items + it);
    x.b0 = e.x; x.ng = e.y; x.row0 = e.z; x.kvh = e.w;
  } else {                                       // (seq, kv head)-major, 256-row chunks
    const int unit = it / p.chunks;
    x.b0 = unit / p.KVH;
    x.kvh = unit - x.b0 * p.KVH;
    x.ng = 1;
    x.row0 = (it - unit * p.chunks) * ROWS;
  }
  x.s_lo = x.row0 / p.Rp;
  const int s_hi = min((x.row0 + ROWS - 1) / p.Rp, x.ng - 1);
  x.n_span = s_hi - x.s_lo + 1;
  int nbc_sum = 0;
#pragma unroll
  for (int k = 0; k < MAX_SPAN; ++k) {
    const int s = x.s_lo + k;
    int nb = 0;
    if (k < x.n_span) {
      // valid local rows of sequence s inside the item; causal: only keys up to
      // the largest token index among them are ever visible
      const int ra = max(x.row0 - s * p.Rp, 0);
      const int rb = min(x.row0 + ROWS - s * p.Rp, p.R) - 1;
      if (ra <= rb) {
        const int t_max = (rb / p.T != ra / p.T) ? p.T - 1 : rb % p.T;
        nb = (t_max + KB) / KB;
      }
    }
    x.nbc[k] = nb;
    nbc_sum += nb;
  }
  x.vlen = p.P ? min(p.prefix_valid_len[x.b0], p.P) : 0;
  x.nb_pre = (x.vlen + KB - 1) / KB;
  x.nb = x.nb_pre + nbc_sum;
  return x;
}
// Suffix block j (>= nb_pre) of an item: which covered sequence, first key.
__device__ __forceinline__ void suffix_block(const Item& x, int j, int& s_rel, int& key0) {
  int jj = j - x.nb_pre, k = 0;
#pragma unroll
  for (int q = 0; q < MAX_SPAN - 1; ++q)
    if (k == q && jj >= x.nbc[q]) { jj -= x.nbc[q]; k = q + 1; }
  s_rel = x.s_lo + k;
  key0 = jj * KB;
}

// Decode one 16-byte chunk of HRKV codes (16 INT8 or 32 INT4, low nibble
// first) into packed 16-bit pairs code * scale.
//
// f16: the codes become exact f16 integers by the magic-number trick (bits
// 0x6400 | u = 1024 + u; INT4 nibbles are masked in place with LOP3, the
// upper nibble of a byte scaled by 1/16 in the same HFMA2) and are multiplied
// by f16 scales with HMUL2 -- ~2 instructions per element, so the two
// converter warps keep up with the MMA/softmax chain.  The result differs from
// krr_dequant_pages' f16(f32 code*scale) by the f16 rounding of the scale
// (<= 2^-11 relative).
// bf16 (no exact magic for 8-bit codes in a bf16 mantissa): f32 2^23 + u,
// FADD, FMUL by the f32 scale, one rounding -- bit-identical to
// krr_dequant_pages.
template <typename T, int QB>
__device__ __forceinline__ void decode_chunk(const uint4 v, const uint32_t* sc, uint32_t* out) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  if constexpr (std::is_same<T, __half>::value) {
    const __half2* s2 = reinterpret_cast<const __half2*>(sc);
    if constexpr (QB == 8) {
      const __half2 bias = __halves2half2(__ushort_as_half(0x6480), __ushort_as_half(0x6480));
#pragma unroll
      for (int i = 0; i < 4; ++i) {                    // 4 codes per word
        const uint32_t wx = w[i] ^ 0x80808080u;       // byte -> code + 128
        const uint32_t lo = __byte_perm(wx, 0x64646464u, 0x4140u);
        const uint32_t hi = __byte_perm(wx, 0x64646464u, 0x4342u);
        const __half2 a = __hmul2(__hsub2(*reinterpret_cast<const __half2*>(&lo), bias), s2[2 * i]);
        const __half2 b = __hmul2(__hsub2(*reinterpret_cast<const __half2*>(&hi), bias),
                                  s2[2 * i + 1]);
        out[2 * i] = *reinterpret_cast<const uint32_t*>(&a);
        out[2 * i + 1] = *reinterpret_cast<const uint32_t*>(&b);
      }
    } else {
      const __half2 b1032 = __halves2half2(__ushort_as_half(0x6408), __ushort_as_half(0x6408));
      const __half2 sixteenth = __halves2half2(__ushort_as_half(0x2C00), __ushort_as_half(0x2C00));
      const __half2 m72 = __halves2half2(__ushort_as_half(0xD480), __ushort_as_half(0xD480));
#pragma unroll
      for (int i = 0; i < 4; ++i) {                    // 8 codes per word: nibble k = channel k
        const uint32_t wx = w[i] ^ 0x88888888u;       // nibble -> code + 8
        const uint32_t wy = wx >> 8;
        uint32_t r[4] = {(wx & 0x000F000Fu) | 0x64006400u, (wx & 0x00F000F0u) | 0x64006400u,
                         (wy & 0x000F000Fu) | 0x64006400u, (wy & 0x00F000F0u) | 0x64006400u};
        __half2 h[4];
        h[0] = __hsub2(*reinterpret_cast<const __half2*>(&r[0]), b1032);                // c0, c4
        h[1] = __hfma2(*reinterpret_cast<const __half2*>(&r[1]), sixteenth, m72);       // c1, c5
        h[2] = __hsub2(*reinterpret_cast<const __half2*>(&r[2]), b1032);                // c2, c6
        h[3] = __hfma2(*reinterpret_cast<const __half2*>(&r[3]), sixteenth, m72);       // c3, c7
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          h[k] = __hmul2(h[k], s2[4 * i + k]);        // scales pre-paired (s_k, s_k+4)
          r[k] = *reinterpret_cast<const uint32_t*>(&h[k]);
        }
        out[4 * i] = __byte_perm(r[0], r[1], 0x5410u);       // c0, c1
        out[4 * i + 1] = __byte_perm(r[2], r[3], 0x5410u);   // c2, c3
        out[4 * i + 2] = __byte_perm(r[0], r[1], 0x7632u);   // c4, c5
        out[4 * i + 3] = __byte_perm(r[2], r[3], 0x7632u);   // c6, c7
      }
    }
  } else {
    const float* sf = reinterpret_cast<const float*>(sc);
    if constexpr (QB == 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t wx = w[i >> 1] ^ 0x80808080u;
        const int b0 = (i & 1) * 2;
        const float f0 = __uint_as_float(__byte_perm(wx, 0x4B000000u, 0x7440u + b0)) - 8388736.f;
        const float f1 = __uint_as_float(__byte_perm(wx, 0x4B000000u, 0x7441u + b0)) - 8388736.f;
        out[i] = pack_2<T>(f0 * sf[2 * i], f1 * sf[2 * i + 1]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t wx = w[i >> 2] ^ 0x88888888u;
        const int sh = (i & 3) * 8;
        const float f0 = __uint_as_float(0x4B000000u | ((wx >> sh) & 0xFu)) - 8388616.f;
        const float f1 = __uint_as_float(0x4B000000u | ((wx >> (sh + 4)) & 0xFu)) - 8388616.f;
        out[i] = pack_2<T>(f0 * sf[2 * i], f1 * sf[2 * i + 1]);
      }
    }
  }
}

// Per-lane scales for decode_chunk: f16 -- half2 pairs in the order the decode
// multiplies (INT8 (s0,s1),(s2,s3)..; INT4 per 8 channels (s0,s4),(s1,s5),
// (s2,s6),(s3,s7)); bf16 -- the f32 scales.
template <typename T, int QB, int CH>
__device__ __forceinline__ void load_scales(const float* src, uint32_t* sc) {
  float f[CH];
  const float4* s4 = reinterpret_cast<const float4*>(src);
#pragma unroll
  for (int i = 0; i < CH / 4; ++i) {
    const float4 v = __ldg(s4 + i);
    f[4 * i] = v.x; f[4 * i + 1] = v.y; f[4 * i + 2] = v.z; f[4 * i + 3] = v.w;
  }
  if constexpr (std::is_same<T, __half>::value) {
#pragma unroll
    for (int k = 0; k < CH / 2; ++k) {
      int a, b;
      if constexpr (QB == 8) { a = 2 * k; b = 2 * k + 1; }
      else { a = (k / 4) * 8 + (k % 4); b = a + 4; }
      __half2 h = __floats2half2_rn(f[a], f[b]);
      sc[k] = *reinterpret_cast<uint32_t*>(&h);
    }
  } else {
#pragma unroll
    for (int k = 0; k < CH; ++k) sc[k] = __float_as_uint(f[k]);
  }
}

template <typename T, int HD, int QB>
__global__ void __launch_bounds__(threads_of<HD, QB>(), 1)
    attn_fa_kernel(const __grid_constant__ CUtensorMap tmQ,
                   const __grid_constant__ CUtensorMap tmPre,
                   const __grid_constant__ CUtensorMap tmCur, const Params p) {
  using S = Smem<HD, QB>;
  constexpr int NT = S::NT;
  constexpr int RK = rk_of<HD, QB>(), RV = rv_of<HD, QB>();
  constexpr int TC = S::TILE_COLS;
  constexpr int NSB = nsb_of<HD>();
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
    for (int i = 0; i < 4; ++i) {
      mbar_init(&bar[B_SFULL + i], 1);
      mbar_init(&bar[B_PFULL + i], 4);
      mbar_init(&bar[B_PVDONE + i], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&bar[B_ODONE + x], 1);
      mbar_init(&bar[B_OEMPTY + x], 4);
    }
    for (int c = 0; c < 2 * NC; ++c) {
      mbar_init(&bar[B_CFULL + c], 1);
      mbar_init(&bar[B_CEMPTY + c], 1);
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
  const int n_items = item_count(p);

  if (warp == 0) {
    // ---------------------------------------------------------- producers
    if (lane == 0) {                                   // Q tiles, per item
      int n = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++n) {
        const Item x = item_of<NT>(p, it);
        mbar_wait(&bar[B_QEMPTY], (n & 1) ^ 1);
        mbar_expect_tx(&bar[B_QFULL], NT * S::Q_TILE);
#pragma unroll
        for (int sub = 0; sub < 2 * NT; ++sub) {            // 64-row boxes, one sequence each
          const int gr = x.row0 + sub * 64;
          int s_rel = gr / p.Rp, r = gr - s_rel * p.Rp;
          if (s_rel >= x.ng) { s_rel = 0; r = 0; }     // past the group: rows unused
          const int unit = (x.b0 + s_rel) * p.KVH + x.kvh;
#pragma unroll
          for (int a = 0; a < HD / 64; ++a)
            tma_load3(sQ + (sub >> 1) * S::Q_TILE + a * S::ATOM_Q + (sub & 1) * 64 * 128, &tmQ,
                      &bar[B_QFULL], a * 64, r, unit);
        }
      }
    } else if (lane < 3) {                             // K ring (lane 1), V ring (lane 2)
      const bool is_k = lane == 1;
      const int nst = is_k ? RK : RV;
      uint64_t* full = &bar[is_k ? B_KFULL : B_VFULL];
      uint64_t* empty = &bar[is_k ? B_KEMPTY : B_VEMPTY];
      uint8_t* ring = is_k ? sK : sV;
      const int cw = is_k ? 0 : 1;
      uint8_t* cring = smem + S::C_OFF + cw * NC * S::CODE_BLK;
      int g = 0, gc = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const Item x = item_of<NT>(p, it);
        const int pre_page = p.P ? (int)((reinterpret_cast<const char*>(p.prefix_kv[x.b0]) -
                                          p.prefix_base) / p.prefix_page_bytes) +
                                       (p.layer * 2) * p.KVH + x.kvh
                                 : 0;
        const int vofs = is_k ? 0 : p.KVH;
        for (int j = 0; j < x.nb; ++j, ++g) {
          const bool pre = j < x.nb_pre;
          if (QB < 16 && pre) {          // codes -> code ring; a converter warp fills K/V
            const int c = gc % NC;
            mbar_wait(&bar[B_CEMPTY + cw * NC + c], ((gc / NC) & 1) ^ 1);
            mbar_expect_tx(&bar[B_CFULL + cw * NC + c], S::CODE_BLK);
            tma_load3(cring + c * S::CODE_BLK, &tmPre, &bar[B_CFULL + cw * NC + c], 0, j * KB,
                      pre_page + vofs);
            ++gc;
            continue;
          }
          const int s = g % nst;
          mbar_wait(&empty[s], ((g / nst) & 1) ^ 1);
          mbar_expect_tx(&full[s], S::KV_BYTES);
          const CUtensorMap* map = pre ? &tmPre : &tmCur;
          int key0 = j * KB, pk = pre_page;
          if (!pre) {
            int s_rel;
            suffix_block(x, j, s_rel, key0);
            pk = (int)((reinterpret_cast<const char*>(p.cur_kv[x.b0 + s_rel]) - p.cur_base) /
                       p.cur_page_bytes) + (p.cur_layer * 2) * p.KVH + x.kvh;
          }
          pk += vofs;
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
    // S_tile(gs) = Q_tile . K(gs)^T into S buffer gs&1
    auto issue_s = [&](int tile, int gs) {
      const int st = gs % RK;
      if (elect_one_sync()) {
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t qoff = tile * S::Q_TILE + (k >> 2) * S::ATOM_Q + (k & 3) * 32;
          const uint32_t koff = st * S::KV_BYTES + (k >> 2) * S::ATOM_KV + (k & 3) * 32;
          mma_f16<1>(tmem + tile * TC + (gs % NSB) * KB, dQ + (qoff >> 4), dK + (koff >> 4),
                     idesc_s, k > 0);
        }
        mma_commit<1>(&bar[B_SFULL + tile * NSB + gs % NSB]);
      }
      __syncwarp();
    };
    // O_tile += P_tile(gs) . V(gs), P in the first KB/2 columns of S buffer gs&1
    auto issue_pv = [&](int tile, int gs, bool acc) {
      const int sv = gs % RV;
      if (elect_one_sync()) {
#pragma unroll
        for (int k = 0; k < KB / 16; ++k)
          mma_ts(tmem + tile * TC + NSB * KB, tmem + tile * TC + (gs % NSB) * KB + k * 8,
                 dV + ((sv * S::KV_BYTES + k * 16 * 128) >> 4), idesc_o, acc || k > 0);
        mma_commit<1>(&bar[B_PVDONE + tile * NSB + gs % NSB]);
      }
      __syncwarp();
    };
    auto issue_s_pair = [&](int gs, bool last_s) {     // S(gs) for both tiles, release K
      mbar_wait(&bar[B_KFULL + gs % RK], (gs / RK) & 1);
      tc_fence_after();
#pragma unroll
      for (int tile = 0; tile < NT; ++tile) issue_s(tile, gs);
      if (elect_one_sync()) {
        mma_commit<1>(&bar[B_KEMPTY + gs % RK]);
        if (last_s) mma_commit<1>(&bar[B_QEMPTY]);      // Q no longer read by this item
      }
      __syncwarp();
    };
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++n) {
      const Item x = item_of<NT>(p, it);
      mbar_wait(&bar[B_QFULL], n & 1);
      for (int j = 0; j < NSB && j < x.nb; ++j) issue_s_pair(g + j, j == x.nb - 1);
      for (int j = 0; j < x.nb; ++j) {
        const int gs = g + j;
        const bool ahead = j + NSB < x.nb;
        TR(2, 4, gs);
        mbar_wait(&bar[B_VFULL + gs % RV], (gs / RV) & 1);
        TR(2, 5, gs);
        if (ahead) mbar_wait(&bar[B_KFULL + (gs + NSB) % RK], ((gs + NSB) / RK) & 1);
        TR(2, 6, gs);
#pragma unroll
        for (int tile = 0; tile < NT; ++tile) {
          if (j == 0) mbar_wait(&bar[B_OEMPTY + tile], (n & 1) ^ 1);
          mbar_wait(&bar[B_PFULL + tile * NSB + gs % NSB], (gs / NSB) & 1);
          TR(2, tile * 2, gs);
          tc_fence_after();
          issue_pv(tile, gs, j > 0);
          if (ahead) issue_s(tile, gs + NSB);   // in-order pipe: PV(gs) reads P before S(gs+NSB) lands
          else if (j == x.nb - 1 && elect_one_sync()) mma_commit<1>(&bar[B_ODONE + tile]);
          __syncwarp();
          TR(2, tile * 2 + 1, gs);
        }
        if (elect_one_sync()) {
          mma_commit<1>(&bar[B_VEMPTY + gs % RV]);
          if (ahead) {
            mma_commit<1>(&bar[B_KEMPTY + (gs + NSB) % RK]);
            if (j + NSB == x.nb - 1) mma_commit<1>(&bar[B_QEMPTY]);
          }
        }
        __syncwarp();
      }
      g += x.nb;
    }
  } else if (warp >= 2 + 4 * NT) {
    // ---------------------------------------------------------- converters (QB < 16)
    if constexpr (QB < 16) {
      const int cw = warp - (2 + 4 * NT);                        // 0: K, 1: V
      uint64_t* full = &bar[cw == 0 ? B_KFULL : B_VFULL];
      uint64_t* empty = &bar[cw == 0 ? B_KEMPTY : B_VEMPTY];
      uint8_t* ring = cw == 0 ? sK : sV;
      const uint8_t* cring = smem + S::C_OFF + cw * NC * S::CODE_BLK;
      constexpr int CPR = S::CODE_ROW / 16;            // 16-byte code chunks per key
      constexpr int CH = 128 / QB;                     // channels per code chunk
      constexpr int RSTEP = 32 / CPR;
      static_assert(CPR >= 1 && CPR <= 32 && KB % RSTEP == 0, "code chunk mapping");
      const int cc = lane % CPR, r0 = lane / CPR;
      uint32_t sc[std::is_same<T, __half>::value ? CH / 2 : CH];
      int g = 0, gc = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const Item x = item_of<NT>(p, it);
        if (x.nb_pre > 0) {
          const int page = (int)((reinterpret_cast<const char*>(p.prefix_kv[x.b0]) -
                                  p.prefix_base) / p.prefix_page_bytes) +
                           (p.layer * 2 + cw) * p.KVH + x.kvh;
          load_scales<T, QB, CH>(p.scales + (int64_t)page * HD + cc * CH, sc);
        }
        for (int j = 0; j < x.nb_pre; ++j, ++gc) {
          const int gg = g + j, s = gg % RK, c = gc % NC;
          mbar_wait(&bar[B_CFULL + cw * NC + c], (gc / NC) & 1);
          mbar_wait(&empty[s], ((gg / RK) & 1) ^ 1);
          const uint8_t* src = cring + c * S::CODE_BLK;
          uint8_t* dst = ring + s * S::KV_BYTES;
#pragma unroll 2
          for (int r = r0; r < KB; r += RSTEP) {
            const uint4 v = *reinterpret_cast<const uint4*>(src + r * S::CODE_ROW + cc * 16);
            uint32_t o[CH / 2];
            decode_chunk<T, QB>(v, sc, o);
#pragma unroll
            for (int oc = 0; oc < CH / 8; ++oc) {      // 8 channels = one 16-byte chunk
              const int ch = cc * CH + oc * 8;
              const int k = (ch & 63) >> 3;
              *reinterpret_cast<uint4*>(dst + (ch >> 6) * S::ATOM_KV + r * 128 +
                                        ((k ^ (r & 7)) << 4)) =
                  make_uint4(o[4 * oc], o[4 * oc + 1], o[4 * oc + 2], o[4 * oc + 3]);
            }
          }
          fence_async_smem();                          // generic writes -> tensor-core reads
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&full[s]);
            mbar_arrive(&bar[B_CEMPTY + cw * NC + c]);
          }
        }
        g += x.nb;
      }
    }
  } else {
    // ---------------------------------------------------------- softmax WGs
    const int tile = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int lrow = quad * 32 + lane;
    const uint32_t lane_base = tmem + tile * TC + ((uint32_t)(quad * 32) << 16);
    const uint32_t o_col = NSB * KB;
    uint64_t* s_full = &bar[B_SFULL + tile * NSB];    // [buf]
    uint64_t* p_full = &bar[B_PFULL + tile * NSB];    // [buf]
    uint64_t* pv_done = &bar[B_PVDONE + tile * NSB];  // [buf]
    const float L2E = 1.4426950408889634f;
    const int T_ = p.T;
    const int H = p.KVH * p.G;
    int g = 0, n = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++n) {
      const Item x = item_of<NT>(p, it);
      const int gr = x.row0 + tile * TM + lrow;       // row in the group's row space
      const int s_row = gr / p.Rp;                     // sequence (relative to b0)
      const int r = gr - s_row * p.Rp;
      const bool row_ok = s_row < x.ng && r < p.R;
      const bool quad_live = __any_sync(0xffffffffu, row_ok);
      const int gq = r / T_, t = r - gq * T_;
      const int b = x.b0 + s_row;
      float m_use = -CUDART_INF_F, l = 0.f;
      for (int j = 0; j < x.nb; ++j) {
        const int gs = g + j, sb = gs % NSB;
        const bool pre = j < x.nb_pre;
        int key0 = j * KB;
        // suffix block (keys of one covered sequence): visible keys as a 64-bit
        // mask -- tok_valid ballot, then causal, none for other sequences' rows
        uint64_t cur_mask = ~0ull;
        if (!pre) {
          int s_blk;
          suffix_block(x, j, s_blk, key0);
          const uint8_t* tv = p.tok_valid + (int64_t)(x.b0 + s_blk) * T_;
          const int k_lo = key0 + lane, k_hi = key0 + 32 + lane;
          const uint32_t lo = __ballot_sync(0xffffffffu, k_lo < T_ && __ldg(tv + k_lo));
          const uint32_t hi = __ballot_sync(0xffffffffu, k_hi < T_ && __ldg(tv + k_hi));
          cur_mask = ((uint64_t)hi << 32) | lo;
          const int rel = t - key0;                     // keys key0+c visible iff c <= rel
          cur_mask &= rel >= 63 ? ~0ull : (rel < 0 ? 0ull : ((2ull << rel) - 1));
          if (s_blk != s_row) cur_mask = 0ull;
        }
        mbar_wait(&s_full[sb], (gs / NSB) & 1);
        if (quad == 2) TR(3 + tile, 0, gs);
        tc_fence_after();
        bool need = false;
        float alpha = 1.f;
        float sv[KB];
        if (quad_live) {
          {
            uint32_t raw[KB / 32][32];
#pragma unroll
            for (int c = 0; c < KB / 32; ++c)
              tmem_ld32_nowait(lane_base + sb * KB + c * 32, raw[c]);
            tmem_ld_wait();
#pragma unroll
            for (int c = 0; c < KB / 32; ++c)
#pragma unroll
              for (int i = 0; i < 32; ++i) sv[c * 32 + i] = __uint_as_float(raw[c][i]);
          }
          if (quad == 2) TR(3 + tile, 1, gs);
          if (!pre) {
#pragma unroll
            for (int c = 0; c < KB; ++c)
              if (!((cur_mask >> c) & 1ull)) sv[c] = -CUDART_INF_F;
          } else if (key0 + KB > x.vlen) {
#pragma unroll
            for (int c = 0; c < KB; ++c)
              if (key0 + c >= x.vlen) sv[c] = -CUDART_INF_F;
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
        if (quad_live && j >= 1 && __any_sync(0xffffffffu, need)) {
          // O must be stable: wait for P.V of block gs-1 (its buffer's barrier)
          mbar_wait(&pv_done[(gs - 1) % NSB], ((gs - 1) / NSB) & 1);
          tc_fence_after();
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
        if (quad == 2) TR(3 + tile, 2, gs);
        if (quad_live) {
          const float neg_m = !row_ok ? -CUDART_INF_F : (m_use == -CUDART_INF_F) ? 0.f : -m_use;
          float l4[4] = {0.f, 0.f, 0.f, 0.f};
          uint32_t w[KB / 2];
#pragma unroll
          for (int i = 0; i < KB / 2; ++i) {
            const float p0 = ex2_approx(fmaf(sv[2 * i], L2E, neg_m));
            const float p1 = ex2_approx(fmaf(sv[2 * i + 1], L2E, neg_m));
            l4[i & 3] += p0 + p1;
            w[i] = pack_2<T>(p0, p1);
          }
          tmem_st32(lane_base + sb * KB, w);          // P over the S columns it came from
          l = l * alpha + ((l4[0] + l4[1]) + (l4[2] + l4[3]));
        }
        tmem_st_wait();
        if (quad == 2) TR(3 + tile, 3, gs);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[sb]);
      }
      // ---------------------------------------------------------- epilogue
      // O / l -> 16-bit rows [b*T + t][(kvh*G + gq)*HD + c].  Each 32-column
      // chunk goes through this warp's staging buffer so that one store
      // instruction writes 8 rows x 64 contiguous bytes (per-row 16 B stores
      // from 32 different rows cost ~14% of the kernel: profiles/r02_attn_ablation.txt)
      mbar_wait(&bar[B_ODONE + tile], n & 1);
      tc_fence_after();
      if (quad_live) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        T* dst = reinterpret_cast<T*>(p.out) + ((int64_t)b * T_ + t) * (H * HD) +
                 (int64_t)(x.kvh * p.G + gq) * HD;
        uint8_t* stg = smem + S::STG_OFF + (warp - 2) * O_STG;
        // the rows this lane stores: rr = i*8 + lane/4, 16 B segment lane%4
        const int seg = lane & 3;
        T* rdst[4];
        bool rok[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int src = i * 8 + (lane >> 2);
          rdst[i] = reinterpret_cast<T*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(dst), src));
          rok[i] = __shfl_sync(0xffffffffu, row_ok, src);
        }
#pragma unroll 1
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t o[32];
          tmem_ld32_nowait(lane_base + o_col + c * 32, o);
          tmem_ld_wait();
          uint4* srow = reinterpret_cast<uint4*>(stg + lane * O_PITCH);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              w[e] = pack_2<T>(__uint_as_float(o[q4 * 8 + 2 * e]) * inv,
                               __uint_as_float(o[q4 * 8 + 2 * e + 1]) * inv);
            srow[q4] = make_uint4(w[0], w[1], w[2], w[3]);
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rr = i * 8 + (lane >> 2);
            if (rok[i])
              reinterpret_cast<uint4*>(rdst[i] + c * 32)[seg] =
                  *reinterpret_cast<const uint4*>(stg + rr * O_PITCH + seg * 16);
          }
          __syncwarp();
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
                  const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box,
                  CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto enc = encoder();
  if (!enc) return fail(KRR_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(map, dt, rank, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(KRR_ECUDA, "attention tensor map encode failed: " + std::to_string((int)r));
  return KRR_OK;
}

template <typename T, int HD, int QB>
static int launch(const AttnParams& a, cudaStream_t s) {
  using Sm = Smem<HD, QB>;
  const CUtensorMapDataType dt = std::is_same<T, __half>::value ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                                : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const int R = a.group * a.seq_len;
  const int Rp = (R + 63) / 64 * 64;                  // rows per sequence in a group
  const int64_t units = (int64_t)a.n_seqs * a.kv_heads;
  constexpr int ROWS = Sm::NT * TM;                   // query rows per work item
  const int chunks = (Rp + ROWS - 1) / ROWS;
  KRR_REQUIRE(a.items == nullptr || a.item_rows == ROWS, KRR_ECONFIG,
              "attention item table built for another item size");
  KRR_REQUIRE(units * R < INT32_MAX && units * (chunks + 1) < INT32_MAX, KRR_ESHAPE,
              "attention batch too large");
  CUtensorMap mq, mp, mc;
  {
    cuuint64_t dims[3] = {(cuuint64_t)HD, (cuuint64_t)R, (cuuint64_t)units};
    cuuint64_t str[2] = {(cuuint64_t)HD * sizeof(T), (cuuint64_t)R * HD * sizeof(T)};
    cuuint32_t box[3] = {64, 64, 1};
    int rc = encode(&mq, a.q, dt, 3, dims, str, box);
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
  // 16-bit pages, or HRKV code pages ([key][HD*QB/8] bytes, no swizzle: the
  // converter warps read them with plain loads)
  const int64_t pre_row = QB == 16 ? (int64_t)HD * sizeof(T) : (int64_t)HD * QB / 8;
  const int64_t pre_page = (int64_t)std::max(a.prefix_len, 1) * pre_row;
  if (QB < 16) {
    KRR_REQUIRE(a.prefix_len > 0 && a.prefix_scales != nullptr, KRR_ECONFIG,
                "quantised prefix pages need prefix_len > 0 and scales");
    cuuint64_t dims[3] = {(cuuint64_t)pre_row, (cuuint64_t)a.prefix_len,
                          (cuuint64_t)(a.prefix_pool_bytes / pre_page)};
    cuuint64_t str[2] = {(cuuint64_t)pre_row, (cuuint64_t)pre_page};
    cuuint32_t box[3] = {(cuuint32_t)pre_row, (cuuint32_t)KB, 1};
    int rc = encode(&mp, a.prefix_pool, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, dims, str, box,
                    CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
  } else if (a.prefix_len > 0) {
    cuuint64_t dims[3] = {(cuuint64_t)HD, (cuuint64_t)a.prefix_len,
                          (cuuint64_t)(a.prefix_pool_bytes / pre_page)};
    cuuint64_t str[2] = {(cuuint64_t)HD * sizeof(T), (cuuint64_t)pre_page};
    cuuint32_t box[3] = {64, (cuuint32_t)KB, 1};
    int rc = encode(&mp, a.prefix_pool, dt, 3, dims, str, box);
    if (rc) return rc;
  } else {
    mp = mc;
  }
  const int implicit = (int)(units * chunks);
  // grouped items: at most one partial chunk per group beyond the rows
  const int64_t bound = a.items ? (int64_t)a.kv_heads *
                                      (((int64_t)a.n_seqs * Rp + ROWS - 1) / ROWS + a.n_seqs)
                                : implicit;
  Params p{a.prefix_kv, static_cast<const char*>(a.prefix_pool), pre_page, a.cur_kv,
           static_cast<const char*>(a.cur_pool), cur_page, a.prefix_valid_len, a.tok_valid,
           a.out, a.prefix_scales, static_cast<const int4*>(a.items), a.n_items, a.kv_heads,
           a.group, a.seq_len, a.prefix_len, a.layer, a.cur_layer, R, Rp, chunks, implicit};
  {
    const int rc = ensure_func_smem((const void*)attn_fa_kernel<T, HD, QB>, Sm::TOTAL);
    if (rc) return rc;
  }
  const int grid = (int)std::min<int64_t>(bound, device_sm_count());
  attn_fa_kernel<T, HD, QB><<<grid, threads_of<HD, QB>(), Sm::TOTAL, s>>>(mq, mp, mc, p);
  return check_launch("attention_fa");
}

// One CTA: sequences sharing a prefix page pointer and adjacent in the batch
// form a group; each group's rows (Rp per sequence) are cut into items of
// `rows` (256, or 128 at head_dim 256), per kv head: items[] = {b0, ng, row0,
// kvh} in (group, kvh, chunk) order, so CTAs running at the same time stream
// the same pages.
__global__ void __launch_bounds__(1024) attn_group_items_kernel(void* const* prefix_kv, int n,
                                                                int Rp, int rows, int KVH,
                                                                int64_t cap, int4* items,
                                                                int* count) {
  __shared__ int wsum[32];
  __shared__ int base;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int b = c0 + threadIdx.x;
    int ng = 0;
    if (b < n && (b == 0 || prefix_kv[b] != prefix_kv[b - 1])) {
      const void* pk = prefix_kv[b];
      ng = 1;
      while (b + ng < n && prefix_kv[b + ng] == pk) ++ng;
    }
    const int ch = ng ? (int)(((int64_t)ng * Rp + rows - 1) / rows) : 0;
    const int cnt = ch * KVH;
    int incl = cnt;                                  // block inclusive scan
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += v;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const int off = base + (wid ? wsum[wid - 1] : 0) + incl - cnt;
    for (int k = 0; k < KVH; ++k)
      for (int c = 0; c < ch; ++c) {
        const int64_t i = off + (int64_t)k * ch + c;
        if (i < cap) items[i] = make_int4(b, ng, c * rows, k);
      }
    __syncthreads();
    if (threadIdx.x == 0) base += wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = (int)((int64_t)base < cap ? (int64_t)base : cap);
}

}  // namespace attn_fa

int attention_item_rows(int head_dim) { return head_dim == 256 ? attn_fa::TM : 2 * attn_fa::TM; }

int64_t attention_items_capacity(int64_t n_seqs, int group, int seq_len, int kv_heads,
                                 int item_rows) {
  const int64_t Rp = ((int64_t)group * seq_len + 63) / 64 * 64;
  return (int64_t)kv_heads * ((n_seqs * Rp + item_rows - 1) / item_rows + n_seqs);
}

int build_attention_items(void* const* prefix_kv, int n_seqs, int group, int seq_len,
                          int kv_heads, int item_rows, void* items, int64_t cap, int* count,
                          cudaStream_t s) {
  const int Rp = (group * seq_len + 63) / 64 * 64;
  KRR_REQUIRE(item_rows == attn_fa::TM || item_rows == 2 * attn_fa::TM, KRR_ECONFIG,
              "attention items are 128 or 256 rows");
  KRR_REQUIRE(cap >= attention_items_capacity(n_seqs, group, seq_len, kv_heads, item_rows) &&
                  cap < INT32_MAX, KRR_ECONFIG, "attention item table too small");
  attn_fa::attn_group_items_kernel<<<1, 1024, 0, s>>>(prefix_kv, n_seqs, Rp, item_rows, kv_heads, cap, static_cast<int4*>(items), count);
  return check_launch("attention_items");
}

#ifdef KRR_PP_TRACE
extern "C" int krr_fa_trace_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, attn_fa::g_fa_trace, sizeof(attn_fa::g_fa_trace)) == cudaSuccess ? 0 : 3;
}
#endif

template <typename T, int QB>
static int launch_hd(const AttnParams& p, cudaStream_t s) {
  if constexpr (QB == 16)
    if (p.head_dim == 256) return attn_fa::launch<T, 256, QB>(p, s);
  return p.head_dim == 64 ? attn_fa::launch<T, 64, QB>(p, s) : attn_fa::launch<T, 128, QB>(p, s);
}

bool attention_tcgen05_supported(int act, const AttnParams& a) {
  return (act == KRR_F16 || act == KRR_BF16) &&
         (a.head_dim == 64 || a.head_dim == 128 || a.head_dim == 256) &&
         a.cur_pool != nullptr && a.cur_pool_bytes > 0 &&
         (a.prefix_len == 0 || (a.prefix_pool != nullptr && a.prefix_pool_bytes > 0));
}

template <typename T, int HD>
static int occupancy(int* out) {
  using Sm = attn_fa::Smem<HD, 16>;
  auto* k = attn_fa::attn_fa_kernel<T, HD, 16>;
  const int rc = ensure_func_smem((const void*)k, Sm::TOTAL);
  if (rc) return rc;
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      out, k, attn_fa::threads_of<HD, 16>(), Sm::TOTAL);
  if (e != cudaSuccess) return fail(KRR_ECUDA, cudaGetErrorString(e));
  return KRR_OK;
}

int attention_tcgen05_occupancy(int act_dtype, int head_dim, int* out) {
  KRR_REQUIRE(head_dim == 64 || head_dim == 128 || head_dim == 256, KRR_EUNSUPPORTED,
              "head_dim 64|128|256");
  if (act_dtype == KRR_BF16)
    return head_dim == 64    ? occupancy<__nv_bfloat16, 64>(out)
           : head_dim == 128 ? occupancy<__nv_bfloat16, 128>(out)
                             : occupancy<__nv_bfloat16, 256>(out);
  return head_dim == 64 ? occupancy<__half, 64>(out)
         : head_dim == 128 ? occupancy<__half, 128>(out)
                           : occupancy<__half, 256>(out);
}

int launch_attention_fa(int act_dtype, const AttnParams& p, cudaStream_t s) {
  if (!attention_tcgen05_supported(act_dtype, p))
    return fail(KRR_EUNSUPPORTED, "TMEM-P attention needs f16/bf16, head_dim 64|128|256 and pool bases");
  const int qb = p.prefix_bits == 0 ? 16 : p.prefix_bits;
  if (qb != 16 && qb != 8 && qb != 4)
    return fail(KRR_ECONFIG, "prefix_bits must be 16 (or 0), 8 or 4");
  if (qb != 16 && p.head_dim > 128)
    return fail(KRR_EUNSUPPORTED, "quantised prefix pages need head_dim 64|128");
  if (act_dtype == KRR_F16) {
    if (qb == 8) return launch_hd<__half, 8>(p, s);
    if (qb == 4) return launch_hd<__half, 4>(p, s);
    return launch_hd<__half, 16>(p, s);
  }
  if (qb == 8) return launch_hd<__nv_bfloat16, 8>(p, s);
  if (qb == 4) return launch_hd<__nv_bfloat16, 4>(p, s);
  return launch_hd<__nv_bfloat16, 16>(p, s);
}

}  // namespace krr
