// GEMM epilogues shared by the tcgen05 and SIMT GEMMs.
//
// A thread owns `n` consecutive accumulator columns (col0 even, n even) of one
// output row.  Semantics follow the reference forward (model.py:365-400):
//   QKV_ROPE : interleaved RoPE on q/k column pairs (model.py:144,370-371),
//              q packed per kv head in (g, t) row order (model.py:377-378),
//              k/v scattered into the sequence's KV slab (layer-major).
//   RESIDUAL : x += acc  (model.py:397, 400)   GELU: tanh GELU (model.py:444-446)
#pragma once
#include "launchers.h"

namespace krr {

template <typename T> struct Pack2;
template <> struct Pack2<float> {
  using V = float2;
  __device__ static inline V make(float a, float b) { return make_float2(a, b); }
};
template <> struct Pack2<__half> {
  using V = __half2;
  __device__ static inline V make(float a, float b) { return __floats2half2_rn(a, b); }
};
template <> struct Pack2<__nv_bfloat16> {
  using V = __nv_bfloat162;
  __device__ static inline V make(float a, float b) { return __floats2bfloat162_rn(a, b); }
};

template <typename T>
__device__ __forceinline__ void store2(T* p, float a, float b) {
  *reinterpret_cast<typename Pack2<T>::V*>(p) = Pack2<T>::make(a, b);
}

template <typename T>
__device__ __forceinline__ void epi_apply(const EpiParams& ep, int64_t row, int col0,
                                          const float* v, int n) {
  if (ep.kind == KRR_EPI_RESIDUAL) {
    float* x = reinterpret_cast<float*>(ep.out) + row * (int64_t)ep.N + col0;
    if ((n & 3) == 0) {
#pragma unroll 4
      for (int j = 0; j < n; j += 4) {
        float4 o = *reinterpret_cast<float4*>(x + j);
        o.x += v[j]; o.y += v[j + 1]; o.z += v[j + 2]; o.w += v[j + 3];
        *reinterpret_cast<float4*>(x + j) = o;
      }
    } else {
      for (int j = 0; j < n; j += 2) {
        float2 o = *reinterpret_cast<float2*>(x + j);
        o.x += v[j]; o.y += v[j + 1];
        *reinterpret_cast<float2*>(x + j) = o;
      }
    }
    return;
  }
  if (ep.kind == KRR_EPI_STORE || ep.kind == KRR_EPI_GELU || ep.kind == KRR_EPI_GLU_GELU ||
      ep.kind == KRR_EPI_GLU_SILU) {   // GLU: v already holds act(gate) * up
    T* o = reinterpret_cast<T*>(ep.out) + row * (int64_t)ep.N + col0;
    const bool g = ep.kind == KRR_EPI_GELU;
#pragma unroll 4
    for (int j = 0; j < n; j += 2) {
      float a = v[j], b = v[j + 1];
      if (g) { a = gelu_tanh(a); b = gelu_tanh(b); }
      store2<T>(o + j, a, b);
    }
    return;
  }
  // KRR_EPI_QKV_ROPE
  const krr_qkv_t& q = ep.qkv;
  const int HD = q.head_dim, H = q.heads, KVH = q.kv_heads, SL = q.seq_len;
  const int G = H / KVH;
  const int64_t b = row / SL;
  const int t = (int)(row - b * SL);
  const int pos = q.positions ? q.positions[row] : q.pos0 + t;
  const float* cs = q.rope_cos + (int64_t)pos * (HD / 2);
  const float* sn = q.rope_sin + (int64_t)pos * (HD / 2);
  for (int j = 0; j < n; j += 2) {
    const int col = col0 + j;
    const int head = col / HD;  // 0..H-1 q, H..H+KVH-1 k, then v
    const int c = col - head * HD;
    float a = v[j], bb = v[j + 1];
    if (head < H + KVH) {
      const float cv = cs[c >> 1], sv = sn[c >> 1];
      const float ra = a * cv - bb * sv;
      const float rb = a * sv + bb * cv;
      a = ra; bb = rb;
    }
    if (head < H) {
      const int kvh = head / G, g = head - kvh * G;
      T* dst = reinterpret_cast<T*>(q.q_out) +
               (((b * KVH + kvh) * G + g) * (int64_t)SL + t) * HD + c;
      store2<T>(dst, a, bb);
    } else {
      const int which = head < H + KVH ? 0 : 1;
      const int kvh = head - H - which * KVH;
      T* slab = reinterpret_cast<T*>(q.kv_seq[b]);
      T* dst = slab + ((int64_t)((q.layer * 2 + which) * KVH + kvh) * q.kv_len + t) * HD + c;
      store2<T>(dst, a, bb);
    }
  }
}

}  // namespace krr
