// Persistent warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[M,N] = A[M,K] . B[N,K]^T    A = activations (16-bit, K-major)
//                                 B = weights [out, in] (16-bit, K-major)
//
// Roles (1 CTA per SM):
//   warp 0      TMA producer: 128B-swizzled A/B tiles into a smem ring
//   warp 1      MMA issuer:   tcgen05.mma.kind::f16, K=16 steps, fp32 accumulators
//                             in TMEM (2 x 256 columns)
//   warps 2..   epilogue:     tcgen05.ld 32x32b.x32 -> fused epilogue -> TMA store
//
// Geometries (a launch's rows decide; all run the same per-element MMA
// sequence, so results are bit-identical across them -- batch invariance):
//   G=1  single CTA, 128 rows x one 256-wide (or narrower) N tile; M <= 128.
//   G=3  cluster of 2 M-adjacent CTAs, 128 rows each; each TMA-loads half of
//        the weight tile and multicasts it into both (L2->SM 32 instead of
//        48 KB per CTA and k-block); double-buffered accumulators, 4 epilogue
//        warps.  Small launches (latency / C2 batches) and > 131k rows.
//   G=8  cuBLAS's geometry: a CTA pair with cta_group::2 M=256 MMAs and 256
//        rows per SM (two pair MMAs per k-step share each stage's B; each SM
//        holds its 128-row half), i.e. A 32 KB + B 16 KB per SM per 8.4 MFLOP
//        instead of 48 KB per 4.2.  The accumulator (2 x 256 columns) is
//        single-buffered, so its two halves are handed over separately: the
//        last 4 k-blocks of a tile run half 0 first, the first 4 of the next
//        tile start half 0 as soon as 8 epilogue warps have drained it.  The
//        power cap grants it ~8% more clock than G=3; launches of 16k-131k
//        rows (32k-row scoring passes) use it.  Other pair variants (one pair
//        MMA per k-step, two pairs sharing the weight by multicast) and a
//        256-row cta_group::1 CTA lost in the step (profiles/r02_gemm_geometry.txt).
//
// Epilogues: RESIDUAL adds the accumulator into the f32 residual stream with a
// TMA bulk reduce-add (cp.reduce.async.bulk.tensor .add, the read-modify-write
// happens in L2 - no read latency in the SM); STORE/GELU write 16-bit tiles
// with TMA bulk stores; QKV_ROPE rotates in registers and scatters q/k/v rows
// with coalesced 16 B stores.  Staging tiles are 128B/64B-swizzled to match
// the tensor maps (bank-conflict free) and double buffered per warp.
//
// The fixed K order per output tile (no split-K) keeps each row's result
// independent of batch composition and of the geometry chosen for a launch
// (SPEC.md:178 batch invariance).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include "epilogue.cuh"
#include "tc_ptx.cuh"

namespace krr {
namespace tc {

constexpr int BN = 256, BK = 64;
constexpr int THREADS = 192;
// G=8 drains each 256-column accumulator half with 8 epilogue warps (two per
// TMEM lane quadrant) so a half is handed back inside the overlap window
template <int G> constexpr int threads_of() { return G == 8 ? 320 : THREADS; }
constexpr int STG_BUF = 4096;                 // one 32x32 chunk (f32) per buffer
constexpr int STG_WARP_BYTES = 2 * STG_BUF;   // double buffered per epilogue warp

template <int G> struct Geo;
template <> struct Geo<1> {
  static constexpr int CS = 1, STAGES = 4, GROUP_M = 16;
  static constexpr int B_ROWS_SMEM = 256;     // rows of the weight tile held per CTA
};
template <> struct Geo<3> {
  static constexpr int CS = 2, STAGES = 4, GROUP_M = 8;
  static constexpr int B_ROWS_SMEM = 256;
};
// G=8 (A/B): CTA pair with cta_group::2 MMAs, 256 rows per SM: two M=256 pair
// MMAs per k-step share each stage's B (each SM holds ITS 128-row half), so an
// SM receives A 32 KB + B 16 KB per 8.4 MFLOP; single-buffered 2 x 256-column
// accumulator per SM.
template <> struct Geo<8> {
  static constexpr int CS = 2, STAGES = 4, GROUP_M = 4;
  static constexpr int B_ROWS_SMEM = 128;
};
template <int G> constexpr int cta_rows() { return G == 8 ? 256 : 128; }
template <int G> constexpr int a_bytes() { return cta_rows<G>() * BK * 2; }
template <int G> constexpr int b_bytes() { return Geo<G>::B_ROWS_SMEM * BK * 2; }
template <int G> constexpr int tile_m() { return cta_rows<G>() * Geo<G>::CS; }   // rows per cluster
template <int G> constexpr int smem_bytes() {
  return Geo<G>::STAGES * (a_bytes<G>() + b_bytes<G>()) + 4 * STG_WARP_BYTES + 1024 /*align*/ +
         512 /*barriers*/;
}

__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// GELU-tanh (model.py:444-446) with the MUFU tanh: its ~2^-11 relative error
// is at the f16 rounding of the stored activation; the f32 debug build keeps tanhf.
// Factored to 5 FP32 ops + 1 MUFU: inner = x * (c0 + c0*0.044715 * x^2),
// 0.5x(1 + t) = h + h*t with h = 0.5x.
__device__ __forceinline__ float gelu_fast(float x) {
  const float x2 = x * x;
  const float inner = x * fmaf(0.0356774081363001f, x2, 0.7978845608028654f);
  const float h = 0.5f * x;
  return fmaf(h, tanh_fast(inner), h);
}

// Raster: GM > 0 -> groups of GM m-tiles sweep all n-tiles (the activation
// panels of a group stay in L2); GM < 0 -> bands of -GM n-tiles sweep all
// m-tiles (a weight band stays in L2 and is read from DRAM once).
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int GM, int& mb,
                                            int& nb) {
  if (GM < 0) {
    const int GN = -GM;
    const int per_band = GN * num_m;
    const int band = tile / per_band;
    const int first_n = band * GN;
    const int bsize = min(num_n - first_n, GN);
    const int r = tile - band * per_band;
    nb = first_n + r % bsize;
    mb = r / bsize;
    return;
  }
  const int per_group = GM * num_n;
  const int group = tile / per_group;
  const int first_m = group * GM;
  const int gsize = min(num_m - first_m, GM);
  const int r = tile - group * per_group;
  mb = first_m + r % gsize;
  nb = r / gsize;
}

template <typename T>
__device__ __forceinline__ uint32_t pack16(float a, float b) {
  typename Pack2<T>::V v = Pack2<T>::make(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ------------------------------------------------------------ QKV row table
// The QKV scatter needs, per output row, its sequence b, token t and (for K/V)
// the sequence's KV page; a tile's 8 chunks share the rows, so each epilogue
// thread resolves them once per tile: its own row (RoPE position) and the four
// rows it stores in the transposed write-out (rr = i*8 + lane/4).
struct QkvRows {
  int pos;              // RoPE position of row row0 + lane
  int b[4], t[4];       // sequence / token of the stored rows (b < 0: past M)
  char* kv[4];          // their sequences' KV pages (kv_seq[b])
};
__device__ __forceinline__ void qkv_rows(const EpiParams& ep, int64_t row0, int lane,
                                         QkvRows& qr) {
  const krr_qkv_t& q = ep.qkv;
  const int SL = q.seq_len;
  const int my = (int)(row0 + lane);                 // M < 2^31 (launch check)
  qr.pos = q.positions ? (my < ep.M ? q.positions[my] : 0) : q.pos0 + my % SL;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = (int)row0 + i * 8 + (lane >> 2);
    const bool ok = row < ep.M;
    const int b = row / SL;
    qr.b[i] = ok ? b : -1;
    qr.t[i] = row - b * SL;
    qr.kv[i] = ok ? reinterpret_cast<char*>(q.kv_seq[b]) : nullptr;
  }
}

// ------------------------------------------------------------ epilogue chunk
// Thread `lane` of an epilogue warp holds row row0+lane, columns col0..col0+31.
template <typename T>
__device__ __forceinline__ void epi_chunk(const EpiParams& ep, const CUtensorMap* out_map,
                                          const uint32_t (&r)[32], int64_t row0, int lane,
                                          int col0, uint8_t* buf, const QkvRows& qr) {
  if (ep.kind == KRR_EPI_RESIDUAL) {
    // f32 chunk, 128B-swizzled rows (16 B piece j of row l at slot j ^ (l & 7))
    uint8_t* row = buf + lane * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<uint4*>(row + ((j ^ (lane & 7)) << 4)) =
          make_uint4(r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_reduce_add(out_map, buf, col0, (int)row0);
      bulk_commit();
    }
    return;
  }
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  if (ep.kind != KRR_EPI_QKV_ROPE) {
    if (ep.kind == KRR_EPI_GELU) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = gelu_fast(v[j]);
    }
    // 16-bit chunk, 64B-swizzled rows (16 B piece j of row l at slot j ^ ((l >> 1) & 3))
    uint8_t* row = buf + lane * 64;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<uint4*>(row + ((j ^ ((lane >> 1) & 3)) << 4)) =
          make_uint4(pack16<T>(v[8 * j], v[8 * j + 1]), pack16<T>(v[8 * j + 2], v[8 * j + 3]),
                     pack16<T>(v[8 * j + 4], v[8 * j + 5]),
                     pack16<T>(v[8 * j + 6], v[8 * j + 7]));
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store(out_map, buf, col0, (int)row0);
      bulk_commit();
    }
    return;
  }
  // QKV: RoPE in registers, then scatter rows of 64 B (4 lanes x 16 B per row).
  const krr_qkv_t& q = ep.qkv;
  const int head = col0 / q.head_dim;
  const int c0 = col0 - head * q.head_dim;
  if (head < q.heads + q.kv_heads) {
    const int64_t off = (int64_t)qr.pos * (q.head_dim / 2) + (c0 >> 1);
    const float4* cp = reinterpret_cast<const float4*>(q.rope_cos + off);
    const float4* sp = reinterpret_cast<const float4*>(q.rope_sin + off);
#pragma unroll
    for (int j4 = 0; j4 < 4; ++j4) {
      const float4 cv = __ldg(cp + j4), sv = __ldg(sp + j4);
      const float cs[4] = {cv.x, cv.y, cv.z, cv.w}, sn[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = (j4 * 4 + u) * 2;
        const float a = v[j], b = v[j + 1];
        v[j] = a * cs[u] - b * sn[u];
        v[j + 1] = a * sn[u] + b * cs[u];
      }
    }
  }
  constexpr int PITCH = 80;  // 64 B row + 16 B pad: conflict-free transpose
  uint4* s = reinterpret_cast<uint4*>(buf + lane * PITCH);
#pragma unroll
  for (int j = 0; j < 4; ++j)
    s[j] = make_uint4(pack16<T>(v[8 * j], v[8 * j + 1]), pack16<T>(v[8 * j + 2], v[8 * j + 3]),
                      pack16<T>(v[8 * j + 4], v[8 * j + 5]), pack16<T>(v[8 * j + 6], v[8 * j + 7]));
  __syncwarp();
  // destination of this chunk's head: q [seq][kvh][g][t][HD] or the sequence's
  // KV page [layer][K|V][kvh][t][HD]; rows then differ only by (b, t)
  const int SL = q.seq_len, HD = q.head_dim, KVH = q.kv_heads, H = q.heads;
  int64_t seq_stride, head_off;
  bool to_q = head < H;
  if (to_q) {
    const int G = H / KVH, kvh = head / G, g = head - kvh * G;
    seq_stride = (int64_t)KVH * G * SL * HD;
    head_off = ((int64_t)(kvh * G + g) * SL) * HD + c0;
  } else {
    const int which = head < H + KVH ? 0 : 1;
    const int kvh = head - H - which * KVH;
    seq_stride = 0;
    head_off = ((int64_t)((q.layer * 2 + which) * KVH + kvh) * q.kv_len) * HD + c0;
  }
  const int seg = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (qr.b[i] >= 0) {
      const int rr = i * 8 + (lane >> 2);
      const uint4 val = *reinterpret_cast<const uint4*>(buf + rr * PITCH + seg * 16);
      T* base = to_q ? reinterpret_cast<T*>(q.q_out) + qr.b[i] * seq_stride
                     : reinterpret_cast<T*>(qr.kv[i]);
      reinterpret_cast<uint4*>(base + head_off + (int64_t)qr.t[i] * HD)[seg] = val;
    }
  }
  __syncwarp();
}

// ------------------------------------------------------------ kernel
template <typename T, int G>
__global__ void __launch_bounds__(threads_of<G>(), 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmOut, int64_t M, int N, int K,
                        uint32_t idesc, int group_m, int bn, EpiParams ep) {
  using C = Geo<G>;
  constexpr int CS = C::CS, STAGES = C::STAGES;
  constexpr int B_BYTES = b_bytes<G>();
  constexpr int A_BYTES = a_bytes<G>();
  constexpr bool PAIR = G == 8;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * A_BYTES;
  uint8_t* stage_base = sB + STAGES * B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_base + 4 * STG_WARP_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CS > 1 ? cluster_rank() : 0;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      // G=3: a stage is free only when BOTH CTAs' MMAs have read it (the peer
      // multicasts its half of B into this CTA's buffer)
      // (pair: one multicast commit of the leader's MMAs frees both CTAs)
      mbar_init(&empty[s], PAIR ? 1 : CS);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], PAIR ? 16 : 4);  // pair: both CTAs' 8 epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(tmem_slot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(tmem_slot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CS > 1) cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_m = (int)((M + tile_m<G>() - 1) / tile_m<G>());
  const int num_n = (N + bn - 1) / bn;
  const int tiles = num_m * num_n;
  const int nk = K / BK;
  const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;

  if (warp == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int tile = cid; tile < tiles; tile += ncl) {
      int mb, nb;
      tile_coords(tile, num_m, num_n, group_m, mb, nb);
      const int row_a = mb * tile_m<G>() + (int)rank * 128;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one_sync()) {
          uint8_t* a_dst = sA + stage * A_BYTES;
          uint8_t* b_dst = sB + stage * B_BYTES;
          if constexpr (PAIR) {
            // both CTAs' bytes complete on the leader's barrier; rows: this SM's
            // 128 of each of the pair tile's two 256-row MMAs, and its B half
            const uint32_t bar = mapa_rank(smem_u32(&full[stage]), 0);
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * (A_BYTES + B_BYTES));
            tma_load<2>(a_dst, &tmA, bar, kb * BK, row_a);
            tma_load<2>(a_dst + 128 * 128, &tmA, bar, kb * BK, row_a + 256);
            tma_load<2>(b_dst, &tmB, bar, kb * BK, nb * bn + (int)rank * 128);
          } else {
          const uint32_t bar = smem_u32(&full[stage]);
          mbar_expect_tx(&full[stage], A_BYTES + bn * BK * 2);
          tma_load<1>(a_dst, &tmA, bar, kb * BK, row_a);
          if constexpr (G == 1) {
            tma_load<1>(b_dst, &tmB, bar, kb * BK, nb * bn);
          } else {
            // own slice of B, multicast into both CTAs' stage buffers
            const int b_rows = bn / 2;
            tma_load_mc(b_dst + rank * (b_rows * BK * 2), &tmB, bar, kb * BK,
                        nb * bn + (int)rank * b_rows, (uint16_t)0x3);
          }
          }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // whole warp walks the schedule; one elected lane issues (descriptors stay
    // in uniform registers, no per-MMA elect loop).  Pair: the leader issues.
    if constexpr (PAIR) {
      if (rank == 0) {
        // Pair schedule with the two 256-column accumulator halves handed over
        // separately: a tile's last `post` k-blocks run MMA#1 (half 0) first so
        // half 0 is committed while MMA#2 finishes; the next tile's first `pre`
        // k-blocks run MMA#1 as soon as half 0 is drained and MMA#2 once half 1
        // is -- each half's epilogue overlaps the other half's MMAs.
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        const uint64_t dA = sw128_desc(smem_u32(sA));
        const uint64_t dB = sw128_desc(smem_u32(sB));
        const int pre = min(STAGES, nk), post = min(STAGES, nk - pre);
        auto mma = [&](int h, int st, int kb) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            mma_f16<2>(tmem_base + h * BN, dA + ((st * A_BYTES + h * 128 * 128 + k * 32) >> 4),
                       dB + ((st * B_BYTES + k * 32) >> 4), idesc, (kb | k) != 0);
        };
        auto adv = [&](int& st, uint32_t& ph) { if (++st == STAGES) { st = 0; ph ^= 1; } };
        for (int tile = cid; tile < tiles; tile += ncl, ++it) {
          const uint32_t ap = it & 1;
          // head: half 0 first, then half 1, on the same resident stages
          mbar_wait(&tempty[0], ap ^ 1);
          tc_fence_after();
          int s0 = stage; uint32_t p0 = phase;
          for (int kb = 0; kb < pre; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (elect_one_sync()) mma(0, stage, kb);
            __syncwarp();
            adv(stage, phase);
          }
          mbar_wait(&tempty[1], ap ^ 1);
          tc_fence_after();
          stage = s0; phase = p0;
          for (int kb = 0; kb < pre; ++kb) {
            if (elect_one_sync()) {
              mma(1, stage, kb);
              mma_commit<2>(&empty[stage]);
            }
            __syncwarp();
            adv(stage, phase);
          }
          // body
          for (int kb = pre; kb < nk - post; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (elect_one_sync()) {
              mma(0, stage, kb);
              mma(1, stage, kb);
              mma_commit<2>(&empty[stage]);
            }
            __syncwarp();
            adv(stage, phase);
          }
          // tail: half 0 completes first
          s0 = stage; p0 = phase;
          for (int kb = nk - post; kb < nk; ++kb) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            if (elect_one_sync()) mma(0, stage, kb);
            __syncwarp();
            adv(stage, phase);
          }
          if (elect_one_sync()) mma_commit<2>(&tfull[0]);
          __syncwarp();
          stage = s0; phase = p0;
          for (int kb = nk - post; kb < nk; ++kb) {
            if (elect_one_sync()) {
              mma(1, stage, kb);
              mma_commit<2>(&empty[stage]);
            }
            __syncwarp();
            adv(stage, phase);
          }
          if (elect_one_sync()) mma_commit<2>(&tfull[1]);
          __syncwarp();
        }
      }
    } else {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      const uint64_t dA = sw128_desc(smem_u32(sA));
      const uint64_t dB = sw128_desc(smem_u32(sB));
      for (int tile = cid; tile < tiles; tile += ncl, ++it) {
        const int acc = it & 1;                         // double-buffered accumulators
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;   // 256 columns apart
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_f16<1>(d_tmem, dA + ((stage * A_BYTES + k * 32) >> 4),
                         dB + ((stage * B_BYTES + k * 32) >> 4), idesc, (kb | k) != 0);
            // completion frees the stage in every CTA that holds its operands
            if constexpr (G == 1) mma_commit<1>(&empty[stage]);
            else mma_commit_mc1(&empty[stage], (uint16_t)0x3);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one_sync()) mma_commit<1>(&tfull[acc]);
        __syncwarp();
      }
    }
  } else {
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    constexpr int EPI = PAIR ? 8 : 4;                  // epilogue warps
    const int sub = (warp - 2) >> 2;                    // pair: which chunk pairs this warp drains
    // pair: one 4 KB staging buffer per warp (8 warps share the 4 x 8 KB area)
    uint8_t* stg = stage_base + (warp - 2) * (PAIR ? STG_BUF : STG_WARP_BYTES);
    int it = 0, nchunk = 0;
    const bool glu = ep.kind == KRR_EPI_GLU_GELU || ep.kind == KRR_EPI_GLU_SILU;
    float gate[32];
    QkvRows qr{};
    for (int tile = cid; tile < tiles; tile += ncl, ++it) {
      int mb, nb;
      tile_coords(tile, num_m, num_n, group_m, mb, nb);
      const int acc = PAIR ? 0 : it & 1;
      const uint32_t acc_phase = PAIR ? it & 1 : (it >> 1) & 1;
      // one epilogue warp polls the accumulator barrier; the other three are
      // parked on a named barrier (the poll loop of four warps was ~1/4 of all
      // issued instructions and power)
      if (warp == 2) mbar_wait(&tfull[acc], acc_phase);
      named_bar_sync(1, 32 * EPI);
      tc_fence_after();
      const int nch = bn / 32;
      const uint32_t tempty_leader = PAIR ? mapa_rank(smem_u32(&tempty[0]), 0) : 0;
#pragma unroll 1
      for (int cc = 0; cc < nch; ++cc) {
        // pair: accumulator h (TMEM columns h*256..) holds rows h*256 + rank*128 ..;
        // this warp drains chunk pairs {4q + 2*sub, +1} of each half
        const int h = PAIR && cc >= nch / 2 ? 1 : 0;
        const int j = cc - h * (nch / 2);
        const int c = PAIR ? (j >> 1) * 4 + sub * 2 + (j & 1) : cc;
        if (PAIR && cc == nch / 2) {
          // half 0 drained: hand it back, then wait for half 1
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_leader);
          if (warp == 2) mbar_wait(&tfull[1], acc_phase);
          named_bar_sync(1, 32 * EPI);
          tc_fence_after();
        }
        const int64_t row0 = (int64_t)mb * tile_m<G>() + h * 256 + rank * 128 + quad * 32;
        if (ep.kind == KRR_EPI_QKV_ROPE && (PAIR ? j == 0 : c == 0)) qkv_rows(ep, row0, lane, qr);
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + (acc + h) * BN + c * 32, r);
        int col0 = nb * bn + c * 32;
        if (col0 >= N) continue;
        if (glu) {
          // even chunk: gate (kept as act(gate)); odd chunk: up -> act(gate) * up
          if (!(c & 1)) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float g = __uint_as_float(r[j]);
              gate[j] = ep.kind == KRR_EPI_GLU_GELU ? gelu_fast(g) : silu(g);
            }
            continue;
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(gate[j] * __uint_as_float(r[j]));
          col0 = (col0 - 32) / 2;
        }
        uint8_t* buf = stg + (PAIR ? 0 : (nchunk & 1) * STG_BUF);
        ++nchunk;
        // the bulk op that last read this buffer (one / two chunks ago) must be done
        if (lane == 0) {
          if constexpr (PAIR) bulk_wait_read<0>();
          else bulk_wait_read<1>();
        }
        __syncwarp();
        epi_chunk<T>(ep, &tmOut, r, row0, lane, col0, buf, qr);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) mbar_arrive_cluster(tempty_leader + 8);   // half 1
        else mbar_arrive(&tempty[acc]);
      }
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CS > 1) cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D row-major [outer, inner] tensor map.
static int make_map(CUtensorMap* map, const void* ptr, CUtensorMapDataType dt, int esize,
                    uint64_t inner, uint64_t outer, uint32_t box_inner, uint32_t box_outer,
                    CUtensorMapSwizzle sw) {
  auto enc = get_encode();
  if (!enc) return fail(KRR_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * (uint64_t)esize};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, dt, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(KRR_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return KRR_OK;
}

template <typename T, int G>
static int launch(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mo, int64_t M,
                  int N, int K, uint32_t idesc, int bn, int group_m, const EpiParams& ep,
                  cudaStream_t s) {
  constexpr int SMEM = smem_bytes<G>();
  {
    const int rc = ensure_func_smem((const void*)gemm_tcgen05_kernel<T, G>, SMEM);
    if (rc) return rc;
  }
  const int tiles = (int)((M + tile_m<G>() - 1) / tile_m<G>()) * ((N + bn - 1) / bn);
  constexpr int CS = Geo<G>::CS;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(threads_of<G>());
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = CS;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  // persistent grid: as many clusters as can be co-resident (GPC boundaries
  // can leave SMs unusable for larger clusters), queried once per device
  const int max_clusters = cached_per_device(
      (const void*)gemm_tcgen05_kernel<T, G>,
      [](const void* c) -> int {
        cudaLaunchConfig_t q = *static_cast<const cudaLaunchConfig_t*>(c);
        q.gridDim = dim3((device_sm_count() / CS) * CS);
        int n = 0;
        if (CS > 1 && cudaOccupancyMaxActiveClusters(&n, gemm_tcgen05_kernel<T, G>, &q) ==
                          cudaSuccess && n > 0)
          return n;
        cudaGetLastError();
        return device_sm_count() / CS;
      },
      &cfg);
  const int grid = std::min(CS * tiles, CS * max_clusters);
  cfg.gridDim = dim3(grid);
  cudaLaunchKernelEx(&cfg, gemm_tcgen05_kernel<T, G>, ma, mb, mo, M, N, K, idesc, group_m, bn, ep);
  return check_launch(G == 1 ? "gemm_tcgen05" : "gemm_tcgen05_mc");
}

}  // namespace tc

int launch_gemm_tcgen05(int act_dtype, const void* A, const void* B, int64_t M, int N, int K,
                        const EpiParams& ep, cudaStream_t s) {
  using namespace tc;
  KRR_REQUIRE(act_dtype == KRR_F16 || act_dtype == KRR_BF16, KRR_EUNSUPPORTED,
              "tcgen05 GEMM needs a 16-bit activation dtype");
  KRR_REQUIRE(K % BK == 0, KRR_ESHAPE, "tcgen05 GEMM needs K % 64 == 0");
  KRR_REQUIRE(N % 32 == 0, KRR_ESHAPE, "tcgen05 GEMM needs N % 32 == 0");
  KRR_REQUIRE(M > 0 && M < (int64_t)INT32_MAX, KRR_ESHAPE, "GEMM M out of range");
  KRR_REQUIRE((reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0,
              KRR_ESHAPE, "GEMM operands must be 16-byte aligned");
  if (ep.kind == KRR_EPI_QKV_ROPE && ep.qkv.head_dim % 32 != 0)
    return launch_gemm_simt(act_dtype, A, B, M, N, K, ep, s);  // a chunk must stay in one head

  // one 128-row tile: a cluster partner would idle.  Launches of 16k-131k rows
  // (the scoring passes of a large batch) take the CTA-pair geometry: it is
  // granted ~8% more clock under the power cap and wins ~0.8% on the C3 step;
  // beyond ~131k rows its loads miss L2 (profiles/r02_gemm_geometry.txt), and
  // small launches need the 128-row units for their wave count.
  const int geo = M <= 128 ? 1 : (M >= 16384 && M <= 131072) ? 8 : 3;
  // N-tile width, chosen by a wave model: each
  // candidate width bn (multiples of 32 so epilogue chunks never straddle a
  // head) gives units = m-tiles x ceil(N/bn) tiles on `slots` persistent
  // CTAs (clusters), cost = ceil(units/slots) waves x bn x c(bn), where
  // c(bn) = 1 + 0.3(256/bn - 1) is the measured per-FLOP penalty of narrower
  // MMAs (A re-read from smem per N-chunk; profiles/r01_gemm_tile_width_sweep.txt:
  // 1.3x at 128).  Large M (thousands of waves) always lands on 256; few-wave
  // launches (the per-query latency batch, C2's N=2048 layers) avoid a
  // mostly-empty last wave.  Every width runs the same per-element MMA
  // sequence (full K in BK-chunk order into one fp32 accumulator), so the
  // choice may depend on M without breaking batch invariance.
  int bn = BN;
  if (geo != 8) {
    const int rows_per_unit = geo == 3 ? 256 : 128;
    const int64_t slots = geo == 3 ? device_sm_count() / 2 : device_sm_count();
    const int64_t m_units = (M + rows_per_unit - 1) / rows_per_unit;
    double best = 0;
    for (int cand = 256; cand >= 64; cand -= 32) {
      const int64_t units = m_units * ((N + cand - 1) / cand);
      const double cost = (double)((units + slots - 1) / slots) * cand * (1.0 + 0.3 * (256.0 / cand - 1.0));
      if (cand == 256 || cost < best * 0.98) { best = cost; bn = cand; }
    }
  }
  const int group_m = geo == 8 ? Geo<8>::GROUP_M : geo == 3 ? Geo<3>::GROUP_M : Geo<1>::GROUP_M;
  const CUtensorMapDataType dt =
      act_dtype == KRR_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap ma, mb, mo;
  int rc = make_map(&ma, A, dt, 2, (uint64_t)K, (uint64_t)M, BK, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  const uint32_t b_box = geo == 1 ? bn : bn / 2;
  rc = make_map(&mb, B, dt, 2, (uint64_t)K, (uint64_t)N, BK, b_box, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  if (ep.kind == KRR_EPI_RESIDUAL) {
    KRR_REQUIRE((reinterpret_cast<uintptr_t>(ep.out) & 15) == 0, KRR_ESHAPE, "residual must be 16-byte aligned");
    rc = make_map(&mo, ep.out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (uint64_t)N, (uint64_t)M, 32, 32,
                  CU_TENSOR_MAP_SWIZZLE_128B);
  } else if (ep.kind == KRR_EPI_STORE || ep.kind == KRR_EPI_GELU || ep.kind == KRR_EPI_GLU_GELU ||
             ep.kind == KRR_EPI_GLU_SILU) {
    KRR_REQUIRE((reinterpret_cast<uintptr_t>(ep.out) & 15) == 0, KRR_ESHAPE, "output must be 16-byte aligned");
    const bool glu = ep.kind == KRR_EPI_GLU_GELU || ep.kind == KRR_EPI_GLU_SILU;
    KRR_REQUIRE(!glu || N % 64 == 0, KRR_ESHAPE, "gated-MLP GEMM needs N % 64 == 0");
    rc = make_map(&mo, ep.out, dt, 2, (uint64_t)(glu ? N / 2 : N), (uint64_t)M, 32, 32,
                  CU_TENSOR_MAP_SWIZZLE_64B);
  } else {
    mo = ma;  // unused by the QKV scatter
  }
  if (rc) return rc;
  // instruction descriptor: D=f32 @4, A/B f16|bf16 @7/@10, K-major both, N>>3 @17, M>>4 @24
  const uint32_t fmt = act_dtype == KRR_BF16 ? 1u : 0u;
  const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(bn >> 3) << 17) |
                         ((uint32_t)((geo == 8 ? 256 : 128) >> 4) << 24);
  if (act_dtype == KRR_F16)
    return geo == 1   ? launch<__half, 1>(ma, mb, mo, M, N, K, idesc, bn, group_m, ep, s)
           : geo == 8 ? launch<__half, 8>(ma, mb, mo, M, N, K, idesc, bn, group_m, ep, s)
                      : launch<__half, 3>(ma, mb, mo, M, N, K, idesc, bn, group_m, ep, s);
  return geo == 1   ? launch<__nv_bfloat16, 1>(ma, mb, mo, M, N, K, idesc, bn, group_m, ep, s)
         : geo == 8 ? launch<__nv_bfloat16, 8>(ma, mb, mo, M, N, K, idesc, bn, group_m, ep, s)
                    : launch<__nv_bfloat16, 3>(ma, mb, mo, M, N, K, idesc, bn, group_m, ep, s);
}

}  // namespace krr
