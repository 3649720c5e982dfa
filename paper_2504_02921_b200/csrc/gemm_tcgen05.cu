// Persistent warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[M,N] = A[M,K] . B[N,K]^T    A = activations (16-bit, K-major)
//                                 B = weights [out, in] (16-bit, K-major)
//
// Roles (192 threads, 1 CTA per SM):
//   warp 0      TMA producer: 128B-swizzled A/B tiles into a smem ring
//   warp 1      MMA issuer:   tcgen05.mma.kind::f16, K=16 steps, fp32 accumulators
//                             in TMEM (2 x 256 columns, double buffered)
//   warps 2..5  epilogue:     tcgen05.ld 32x32b.x32 -> fused epilogue -> TMA store
//
// Every CTA owns 128 output rows x one 256-wide (or narrower) N tile; the
// geometries differ in how the weight tile reaches the tensor cores:
//   G=1  single CTA, cta_group::1 M=128 MMAs; the CTA loads its whole B tile.
//   G=3  cluster of 2 M-adjacent CTAs, cta_group::1 MMAs; each CTA TMA-loads
//        half of B and multicasts it into both CTAs.  L2->SM 32 KB per CTA and
//        k-block, 48 KB written into each CTA's smem and read by its MMAs.
//   G=7  (default for large M) cluster of 4 = two CTA pairs on M-adjacent
//        256-row tiles sharing the weight tile.  Each pair runs cta_group::2
//        M=256 MMAs issued by its leader: every SM holds only ITS half of B
//        (the pair MMA reads both halves), and that half arrives as two 64-row
//        pieces, one loaded by this CTA and one by the same-half CTA of the
//        other pair, each multicast into both.  Per CTA and k-block: 24 KB read
//        from L2, 32 KB written into smem, 32 KB of operands read by the
//        tensor cores (G=3: 32 / 48 / 48) -- operand movement is what the
//        power cap charges for (profiles/r02_gemm_geometry.txt).
//   G=2  one CTA pair (cluster of 2) without the cross-pair multicast (A/B).
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

// A/B switch for the pair geometries: 1 = plain TMA per CTA + a relayed
// "stage landed" arrive to the pair leader instead of cta_group::2 TMA.
#ifndef KRR_PAIR_RELAY
#define KRR_PAIR_RELAY 0
#endif

namespace krr {
namespace tc {

constexpr int BN = 256, BK = 64;
constexpr int THREADS = 192;
constexpr int STG_BUF = 4096;                 // one 32x32 chunk (f32) per buffer
constexpr int STG_WARP_BYTES = 2 * STG_BUF;   // double buffered per epilogue warp

template <int G> struct Geo;
template <> struct Geo<1> {
  static constexpr int CS = 1, MMA_CG = 1, STAGES = 4, GROUP_M = 16;
  static constexpr int B_ROWS_SMEM = 256;     // rows of the weight tile held per CTA
};
template <> struct Geo<3> {
  static constexpr int CS = 2, MMA_CG = 1, STAGES = 4, GROUP_M = 8;
  static constexpr int B_ROWS_SMEM = 256;
};
template <> struct Geo<2> {
  static constexpr int CS = 2, MMA_CG = 2, STAGES = 6, GROUP_M = 8;
  static constexpr int B_ROWS_SMEM = 128;
};
template <> struct Geo<7> {
  static constexpr int CS = 4, MMA_CG = 2, STAGES = 6, GROUP_M = 4;
  static constexpr int B_ROWS_SMEM = 128;
};
constexpr int A_BYTES = 128 * BK * 2;                      // 16 KB: 128 rows per CTA
template <int G> constexpr int b_bytes() { return Geo<G>::B_ROWS_SMEM * BK * 2; }
template <int G> constexpr int tile_m() { return 128 * Geo<G>::CS; }   // rows per cluster
template <int G> constexpr int smem_bytes() {
  return Geo<G>::STAGES * (A_BYTES + b_bytes<G>()) + 4 * STG_WARP_BYTES + 1024 /*align*/ +
         512 /*barriers*/;
}

__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// GELU-tanh (model.py:444-446) with the MUFU tanh: its ~2^-11 relative error
// is at the f16 rounding of the stored activation; the f32 debug build keeps tanhf.
__device__ __forceinline__ float gelu_fast(float x) {
  const float inner = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  return 0.5f * x * (1.0f + tanh_fast(inner));
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

// ------------------------------------------------------------ epilogue chunk
// Thread `lane` of an epilogue warp holds row row0+lane, columns col0..col0+31.
template <typename T>
__device__ __forceinline__ void epi_chunk(const EpiParams& ep, const CUtensorMap* out_map,
                                          const uint32_t (&r)[32], int64_t row0, int lane,
                                          int col0, uint8_t* buf) {
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
  const int64_t M = ep.M;
  const int head = col0 / q.head_dim;
  const int c0 = col0 - head * q.head_dim;
  if (head < q.heads + q.kv_heads) {
    const int64_t my_row = row0 + lane;
    const int pos = q.positions ? (my_row < M ? q.positions[my_row] : 0)
                                : q.pos0 + (int)(my_row % q.seq_len);
    const int64_t off = (int64_t)pos * (q.head_dim / 2) + (c0 >> 1);
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
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rr = i * 8 + (lane >> 2), seg = lane & 3;
    const int64_t row = row0 + rr;
    if (row < M) {
      const uint4 val = *reinterpret_cast<const uint4*>(buf + rr * PITCH + seg * 16);
      const int SL = q.seq_len, HD = q.head_dim, KVH = q.kv_heads, H = q.heads;
      const int64_t b = row / SL;
      const int t = (int)(row - b * SL);
      T* dst;
      if (head < H) {
        const int G = H / KVH, kvh = head / G, g = head - kvh * G;
        dst = reinterpret_cast<T*>(q.q_out) + (((b * KVH + kvh) * G + g) * (int64_t)SL + t) * HD + c0;
      } else {
        const int which = head < H + KVH ? 0 : 1;
        const int kvh = head - H - which * KVH;
        dst = reinterpret_cast<T*>(q.kv_seq[b]) +
              ((int64_t)((q.layer * 2 + which) * KVH + kvh) * q.kv_len + t) * HD + c0;
      }
      reinterpret_cast<uint4*>(dst)[seg] = val;
    }
  }
  __syncwarp();
}

// ------------------------------------------------------------ kernel
template <typename T, int G>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmOut, int64_t M, int N, int K,
                        uint32_t idesc, int group_m, int bn, EpiParams ep) {
  using C = Geo<G>;
  constexpr int CS = C::CS, MMA_CG = C::MMA_CG, STAGES = C::STAGES;
  constexpr int B_BYTES = b_bytes<G>();
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
  uint64_t* peer_full = tempty + 2;          // RELAY: peer's stage landed (leader side)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(peer_full + STAGES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CS > 1 ? cluster_rank() : 0;
  // cta_group::2: the pair is (rank & ~1, rank | 1); its even CTA leads
  const uint32_t pair_leader = MMA_CG == 2 ? (rank & ~1u) : rank;
  const bool leader = rank == pair_leader;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&peer_full[s], 1);
      // a stage may be refilled once every MMA issuer that reads it committed:
      // G=3 both CTAs (the peer's B slice lands here), G=7 both pair leaders
      // (the other pair multicasts a B piece here), else this CTA's (pair's)
      mbar_init(&empty[s], G == 3 ? 2 : G == 7 ? 2 : 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * MMA_CG);    // every epilogue warp of the pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (MMA_CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(tmem_slot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                       smem_u32(tmem_slot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
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
          if constexpr (G == 1) {
            const uint32_t bar = smem_u32(&full[stage]);
            mbar_expect_tx(&full[stage], A_BYTES + bn * BK * 2);
            tma_load<1>(a_dst, &tmA, bar, kb * BK, row_a);
            tma_load<1>(b_dst, &tmB, bar, kb * BK, nb * bn);
          } else if constexpr (G == 3) {
            // own A rows; own slice of B multicast into both CTAs' stage buffers
            const int b_rows = bn / 2;
            const uint32_t bar = smem_u32(&full[stage]);
            mbar_expect_tx(&full[stage], A_BYTES + bn * BK * 2);
            tma_load<1>(a_dst, &tmA, bar, kb * BK, row_a);
            tma_load_mc(b_dst + rank * (b_rows * BK * 2), &tmB, bar, kb * BK,
                        nb * bn + (int)rank * b_rows, (uint16_t)0x3);
          } else if constexpr (KRR_PAIR_RELAY) {
            // pair, relayed: plain TMA into this CTA's own stage and barrier; the
            // peer's warp 1 forwards "landed" to the leader (peer_full)
            const uint32_t bar = smem_u32(&full[stage]);
            mbar_expect_tx(&full[stage], A_BYTES + B_BYTES);
            tma_load<1>(a_dst, &tmA, bar, kb * BK, row_a);
            const int half = (int)(rank & 1);
            if constexpr (G == 2) {
              tma_load<1>(b_dst, &tmB, bar, kb * BK, nb * bn + half * 128);
            } else {
              const int p = (int)(rank >> 1);
              tma_load_mc(b_dst + p * (64 * BK * 2), &tmB, bar, kb * BK,
                          nb * bn + half * 128 + p * 64, (uint16_t)((1u << rank) | (1u << (rank ^ 2))));
            }
          } else {
            // pair: every byte of both CTAs' stage lands on the pair leader's barrier
            const uint32_t bar = mapa_rank(smem_u32(&full[stage]), pair_leader);
            if (leader) mbar_expect_tx(&full[stage], 2 * (A_BYTES + B_BYTES));
            tma_load<2>(a_dst, &tmA, bar, kb * BK, row_a);
            const int half = (int)(rank & 1);          // which 128-row half of the N tile
            if constexpr (G == 2) {
              tma_load<2>(b_dst, &tmB, bar, kb * BK, nb * bn + half * 128);
            } else {
              // piece p (64 rows) of this half, multicast into the same-half CTA of both pairs
              const int p = (int)(rank >> 1);
              tma_load_mc2(b_dst + p * (64 * BK * 2), &tmB, bar, kb * BK,
                           nb * bn + half * 128 + p * 64, (uint16_t)((1u << rank) | (1u << (rank ^ 2))));
            }
          }
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // whole warp walks the schedule; one elected lane issues (descriptors stay
    // in uniform registers); pair geometries: the leader issues for both SMs
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      const uint64_t dA = sw128_desc(smem_u32(sA));
      const uint64_t dB = sw128_desc(smem_u32(sB));
      // completion of a stage's MMAs frees it in every CTA that holds its operands
      constexpr uint16_t EMPTY_MASK = G == 3 ? 0x3 : G == 7 ? 0xF : 0x0;
      const uint16_t pair_mask = (uint16_t)(0x3u << rank);   // (leader, peer)
      for (int tile = cid; tile < tiles; tile += ncl, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;   // accumulators 256 columns apart
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          if constexpr (MMA_CG == 2 && KRR_PAIR_RELAY) mbar_wait(&peer_full[stage], phase);
          tc_fence_after();
          if (elect_one_sync()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_f16<MMA_CG>(d_tmem, dA + ((stage * A_BYTES + k * 32) >> 4),
                              dB + ((stage * B_BYTES + k * 32) >> 4), idesc, (kb | k) != 0);
            if constexpr (G == 1) mma_commit<1>(&empty[stage]);
            else if constexpr (G == 3) mma_commit_mc1(&empty[stage], EMPTY_MASK);
            else if constexpr (G == 2) mma_commit2_mc(&empty[stage], pair_mask);
            else mma_commit2_mc(&empty[stage], EMPTY_MASK);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one_sync()) {
          if constexpr (MMA_CG == 1) mma_commit<1>(&tfull[acc]);
          else mma_commit2_mc(&tfull[acc], pair_mask);
        }
        __syncwarp();
      }
    } else if constexpr (MMA_CG == 2 && KRR_PAIR_RELAY) {
      // the peer's idle MMA warp relays each landed stage to the leader
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t lead_pf = mapa_rank(smem_u32(&peer_full[0]), pair_leader);
      for (int tile = cid; tile < tiles; tile += ncl)
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          if (elect_one_sync()) mbar_arrive_cluster(lead_pf + stage * 8);
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
    }
  } else {
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    uint8_t* stg = stage_base + (warp - 2) * STG_WARP_BYTES;
    const uint32_t tempty0 = MMA_CG == 2 ? mapa_rank(smem_u32(&tempty[0]), pair_leader)
                                         : smem_u32(&tempty[0]);
    int it = 0, nchunk = 0;
    const bool glu = ep.kind == KRR_EPI_GLU_GELU || ep.kind == KRR_EPI_GLU_SILU;
    float gate[32];
    for (int tile = cid; tile < tiles; tile += ncl, ++it) {
      int mb, nb;
      tile_coords(tile, num_m, num_n, group_m, mb, nb);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      // one epilogue warp polls the accumulator barrier; the other three are
      // parked on a named barrier (the poll loop of four warps was ~1/4 of all
      // issued instructions and power)
      if (warp == 2) mbar_wait(&tfull[acc], acc_phase);
      named_bar_sync(1, 128);
      tc_fence_after();
      const int64_t row0 = (int64_t)mb * tile_m<G>() + rank * 128 + quad * 32;
#pragma unroll 1
      for (int c = 0; c < bn / 32; ++c) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN + c * 32, r);
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
        uint8_t* buf = stg + (nchunk & 1) * STG_BUF;
        ++nchunk;
        // the bulk op that last read this buffer (two chunks ago) must be done
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        epi_chunk<T>(ep, &tmOut, r, row0, lane, col0, buf);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
    }
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CS > 1) cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (MMA_CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
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
  cfg.blockDim = dim3(THREADS);
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
  return check_launch(G == 7 ? "gemm_tcgen05_pair_mc" : G == 2 ? "gemm_tcgen05_pair"
                      : G == 3 ? "gemm_tcgen05_mc" : "gemm_tcgen05");
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

  // Geometry per launch (KRR_GEMM_GEO overrides for A/B: 1, 2, 3 or 7):
  //   M <= 128          G=1 (a cluster partner would idle)
  //   large M           G=7 (pair MMAs + cross-pair weight multicast)
  //   otherwise         G=3
  static const int env_geo = [] {
    const char* e = getenv("KRR_GEMM_GEO");
    const int v = e ? atoi(e) : 0;
    return (v == 1 || v == 2 || v == 3 || v == 7) ? v : 0;
  }();
  int geo = env_geo ? env_geo : (M <= 128 ? 1 : 3);
  if (geo == 1 && M > 128 && env_geo == 0) geo = 3;
  // N-tile width for the cta_group::1 geometries, chosen by a wave model: each
  // candidate width bn (multiples of 32 so epilogue chunks never straddle a
  // head) gives units = m-tiles x ceil(N/bn) tiles on `slots` persistent
  // CTAs (clusters), cost = ceil(units/slots) waves x bn x c(bn), where
  // c(bn) = 1 + 0.3(256/bn - 1) is the measured per-FLOP penalty of narrower
  // MMAs (A re-read from smem per N-chunk; profiles/r01_gemm_tile_width_sweep.txt:
  // 1.3x at 128).  Large M (thousands of waves) always lands on 256; few-wave
  // launches (the per-query latency batch, C2's N=2048 layers) avoid a
  // mostly-empty last wave.  Every width runs the same per-element MMA
  // sequence (full K in BK-chunk order into one fp32 accumulator), so the
  // choice may depend on M without breaking batch invariance.  The pair
  // geometries keep 256 (their B halves are 128 rows).
  int bn = BN;
  if (geo == 1 || geo == 3) {
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
  static const int env_gm = [] {
    const char* e = getenv("KRR_GEMM_GROUP_M");
    return e ? atoi(e) : 0;
  }();
  int group_m = env_gm != 0 ? env_gm          // < 0: bands of -env_gm n-tiles
                : geo == 7 ? Geo<7>::GROUP_M : geo == 2 ? Geo<2>::GROUP_M
                : geo == 3 ? Geo<3>::GROUP_M : Geo<1>::GROUP_M;
  if (env_gm == 0 && (geo == 2 || geo == 7)) {
    // pair geometries: keep the weights L2-resident and stream activations --
    // the whole weight matrix when it fits (QKV, WO: all n-tiles in one band),
    // else bands of 16 n-tiles when those fit (MLP-up), else M-groups (MLP-down)
    const double wbytes = (double)N * K * 2;
    const int num_n = (N + bn - 1) / bn;
    if (wbytes <= 64.0 * (1 << 20)) group_m = -num_n;
    else if (16.0 * bn * K * 2 <= 40.0 * (1 << 20)) group_m = -16;
  }
  const CUtensorMapDataType dt =
      act_dtype == KRR_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap ma, mb, mo;
  int rc = make_map(&ma, A, dt, 2, (uint64_t)K, (uint64_t)M, BK, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  const uint32_t b_box = geo == 1 ? bn : geo == 3 ? bn / 2 : geo == 2 ? 128 : 64;
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
  const int mma_m = (geo == 2 || geo == 7) ? 256 : 128;
  const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(bn >> 3) << 17) |
                         ((uint32_t)(mma_m >> 4) << 24);
#define KRR_GEO_LAUNCH(T)                                                             \
  switch (geo) {                                                                      \
    case 1: return launch<T, 1>(ma, mb, mo, M, N, K, idesc, bn, group_m, ep, s);      \
    case 2: return launch<T, 2>(ma, mb, mo, M, N, K, idesc, bn, group_m, ep, s);      \
    case 7: return launch<T, 7>(ma, mb, mo, M, N, K, idesc, bn, group_m, ep, s);      \
    default: return launch<T, 3>(ma, mb, mo, M, N, K, idesc, bn, group_m, ep, s);     \
  }
  if (act_dtype == KRR_F16) { KRR_GEO_LAUNCH(__half) }
  KRR_GEO_LAUNCH(__nv_bfloat16)
#undef KRR_GEO_LAUNCH
}

}  // namespace krr
