// C ABI entry points (include/kvrerank_b200.h), small kernels, and the
// layer-loop driver krr_forward.
#include <math_constants.h>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>
#include "launchers.h"

namespace krr {

static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& m) { g_err = m; }
int fail(int code, const std::string& m) {
  g_err = m;
  return code;
}
std::atomic<uint64_t>& launch_counter() { return g_launches; }
int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(KRR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return KRR_OK;
}

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

static std::mutex g_dev_mu;
static std::map<std::pair<int, const void*>, int> g_dev_cache;

int cached_per_device(const void* key, int (*compute)(const void*), const void* ctx) {
  const auto k = std::make_pair(current_device(), key);
  {
    std::lock_guard<std::mutex> g(g_dev_mu);
    auto it = g_dev_cache.find(k);
    if (it != g_dev_cache.end()) return it->second;
  }
  const int v = compute(ctx);          // outside the lock: may call into the runtime
  std::lock_guard<std::mutex> g(g_dev_mu);
  return g_dev_cache.emplace(k, v).first->second;
}

static int sm_count_of(const void*) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, current_device());
  return n > 0 ? n : 148;
}

int device_sm_count() {
  static const char key = 0;
  return cached_per_device(&key, sm_count_of, nullptr);
}

struct SmemReq { const void* func; int bytes, carveout; };
static int apply_smem(const void* ctx) {
  const SmemReq* r = static_cast<const SmemReq*>(ctx);
  cudaError_t e = cudaFuncSetAttribute(r->func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       r->bytes);
  if (e == cudaSuccess && r->carveout >= 0)
    e = cudaFuncSetAttribute(r->func, cudaFuncAttributePreferredSharedMemoryCarveout,
                             r->carveout);
  return e == cudaSuccess ? r->bytes : -(int)e;
}

int ensure_func_smem(const void* func, int smem_bytes, int carveout) {
  SmemReq r{func, smem_bytes, carveout};
  // keyed by the function (+1: other per-device values keyed by the same kernel
  // use the plain pointer); a kernel's smem size is a compile-time constant
  const int v = cached_per_device(static_cast<const char*>(func) + 1, apply_smem, &r);
  if (v < 0) return fail(KRR_ECUDA, std::string("cudaFuncSetAttribute failed: ") +
                                        cudaGetErrorString((cudaError_t)(-v)));
  return KRR_OK;
}

// ---------------------------------------------------------------- profiling
struct ProfRec { cudaEvent_t a, b; int cls; double flops; };
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static double g_prof_ms[3] = {0, 0, 0};
static uint64_t g_prof_n[3] = {0, 0, 0};
static double g_prof_flops = 0.0;

ProfScope::ProfScope(cudaStream_t s_, int cls_, double flops_)
    : s(s_), cls(cls_), flops(flops_), on(g_prof_on) {
  if (on) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
}
ProfScope::~ProfScope() {
  if (on) {
    cudaEventRecord(e1, s);
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof.push_back({e0, e1, cls, flops});
  }
}

// ---------------------------------------------------------------- kernels
// a1: SplitMix64 stream -> top 24 bits -> [-b, b] (hashing.py:58-80), written
// in destination order; transpose maps reference [in,out] to device [out,in].
template <typename T>
__global__ void init_uniform_kernel(uint64_t seed, double bound, int64_t rows, int64_t cols,
                                    int transpose, T* out, int64_t ld) {
  const int64_t total = rows * cols;
  for (int64_t d = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; d < total;
       d += (int64_t)gridDim.x * blockDim.x) {
    int64_t r, c, src;
    if (transpose) { c = d / rows; r = d - c * rows; }
    else { r = d / cols; c = d - r * cols; }
    src = r * cols + c;
    uint64_t z = seed + (uint64_t)(src + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    const double u = (double)(z >> 40) / 16777215.0;
    const double two_u = 2.0 * u;                  // exact
    const float v = (float)(__dsub_rn(two_u, 1.0) * bound);
    const int64_t dst = transpose ? c * ld + r : r * ld + c;
    out[dst] = Act<T>::from(v);
  }
}

// a5: x = E[tokens]  (model.py:352)
__global__ void embed_kernel(const int32_t* __restrict__ tok, const float* __restrict__ emb,
                             int d, float scale, float* __restrict__ x) {
  const int64_t r = blockIdx.x;
  const float4* src = reinterpret_cast<const float4*>(emb + (int64_t)tok[r] * d);
  float4* dst = reinterpret_cast<float4*>(x + r * d);
  if (scale == 1.0f) {
    for (int i = threadIdx.x; i < d / 4; i += blockDim.x) dst[i] = src[i];
  } else {   // Gemma-style embedding scale (architecture variant)
    for (int i = threadIdx.x; i < d / 4; i += blockDim.x) {
      const float4 v = src[i];
      dst[i] = make_float4(v.x * scale, v.y * scale, v.z * scale, v.w * scale);
    }
  }
}

static int launch_embed(const int32_t* tokens, const float* emb, int64_t rows, int32_t d,
                        float scale, float* x, cudaStream_t s) {
  KRR_REQUIRE(d % 4 == 0, KRR_ESHAPE, "model_dim must be a multiple of 4");
  if (rows == 0) return KRR_OK;
  ProfScope ps(s, 2);
  embed_kernel<<<(unsigned)rows, 128, 0, s>>>(tokens, emb, d, scale, x);
  return check_launch("embed");
}

// F (MLP width) and the up-projection's GEMM width / epilogue for a model
static inline int ffn_of(const krr_model_t* m) {
  return m->ffn_dim > 0 ? m->ffn_dim : 4 * m->model_dim;
}

__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  if (threadIdx.x < 32) {
    t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// RMSNorm x * (1/sqrt(mean(x^2)+1e-6)) * gain  (model.py:439-441)
template <typename T>
__global__ void rmsnorm_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                               int d, T* __restrict__ out) {
  __shared__ float red[32];
  const int64_t r = blockIdx.x;
  const float* xr = x + r * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss = fmaf(xr[i], xr[i], ss);
  ss = block_sum(ss, red);
  const float inv = 1.0f / sqrtf(ss / (float)d + 1e-6f);
  T* o = out + r * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) o[i] = Act<T>::from((xr[i] * inv) * gain[i]);
}

// Vectorised single-pass RMSNorm: the row stays in registers (VPT float4 per
// thread), one block-reduction, 16-bit output written as 8-byte vectors.
template <typename T, int VPT>
__global__ void rmsnorm_vec_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                                   int d, T* __restrict__ out) {
  __shared__ float red[32];
  const int64_t r = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + r * d);
  const float4* gr = reinterpret_cast<const float4*>(gain);
  float4 v[VPT];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    v[i] = __ldcs(xr + threadIdx.x + i * blockDim.x);
    ss = fmaf(v[i].x, v[i].x, ss); ss = fmaf(v[i].y, v[i].y, ss);
    ss = fmaf(v[i].z, v[i].z, ss); ss = fmaf(v[i].w, v[i].w, ss);
  }
  ss = block_sum(ss, red);
  const float inv = 1.0f / sqrtf(ss / (float)d + 1e-6f);
  T* o = out + r * d;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int e = threadIdx.x + i * blockDim.x;
    const float4 g = __ldg(gr + e);
    const float a = (v[i].x * inv) * g.x, b = (v[i].y * inv) * g.y;
    const float c = (v[i].z * inv) * g.z, dd = (v[i].w * inv) * g.w;
    if constexpr (sizeof(T) == 4) {
      reinterpret_cast<float4*>(o)[e] = make_float4(a, b, c, dd);
    } else {
      T h[4] = {Act<T>::from(a), Act<T>::from(b), Act<T>::from(c), Act<T>::from(dd)};
      reinterpret_cast<uint2*>(o)[e] = *reinterpret_cast<uint2*>(h);
    }
  }
}

// a10: score = rms(x[last])*final_gain . head  (model.py:402, reranker.py:211-212)
__global__ void score_kernel(const float* __restrict__ x, int T_, int d,
                             const int32_t* __restrict__ last, const float* __restrict__ fg,
                             const float* __restrict__ head, float* __restrict__ scores) {
  __shared__ float red[32];
  const int b = blockIdx.x;
  const float* xr = x + ((int64_t)b * T_ + (last ? last[b] : 0)) * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss = fmaf(xr[i], xr[i], ss);
  ss = block_sum(ss, red);
  const float inv = 1.0f / sqrtf(ss / (float)d + 1e-6f);
  float dot = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) dot = fmaf((xr[i] * inv) * fg[i], head[i], dot);
  dot = block_sum(dot, red);
  if (threadIdx.x == 0) scores[b] = dot;
}

// Gather the scored row of every sequence: dst[b] = src[b*T + last[b]]
// (width elements of E bytes), so the last layer's WO/MLP run on n rows only.
template <typename E>
__global__ void gather_last_kernel(const E* __restrict__ src, const int32_t* __restrict__ last,
                                   int T_, int width, E* __restrict__ dst) {
  const int b = blockIdx.x;
  const E* s = src + ((int64_t)b * T_ + last[b]) * width;
  E* o = dst + (int64_t)b * width;
  for (int i = threadIdx.x; i < width; i += blockDim.x) o[i] = s[i];
}

// a13: per-segment top-k by (score desc, doc id asc) (pipeline.py:285-287).
// Rank of candidate i = #{j : s_j > s_i or (s_j == s_i and id_j < id_i)}.
__global__ void topk_kernel(const float* __restrict__ scores, const int32_t* __restrict__ ids,
                            int seg_len, int k, int32_t* __restrict__ out_idx,
                            float* __restrict__ out_score) {
  extern __shared__ uint8_t sm[];
  float* s = reinterpret_cast<float*>(sm);
  int32_t* id = reinterpret_cast<int32_t*>(s + seg_len);
  const int seg = blockIdx.x;
  for (int i = threadIdx.x; i < seg_len; i += blockDim.x) {
    s[i] = scores[(int64_t)seg * seg_len + i];
    id[i] = ids[(int64_t)seg * seg_len + i];
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    out_idx[(int64_t)seg * k + i] = -1;
    if (out_score) out_score[(int64_t)seg * k + i] = -CUDART_INF_F;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < seg_len; i += blockDim.x) {
    const float si = s[i];
    const int32_t ii = id[i];
    int rank = 0;
    for (int j = 0; j < seg_len; ++j) {
      const float sj = s[j];
      rank += (sj > si) || (sj == si && id[j] < ii) || (sj == si && id[j] == ii && j < i);
    }
    if (rank < k) {
      out_idx[(int64_t)seg * k + rank] = i;
      if (out_score) out_score[(int64_t)seg * k + rank] = si;
    }
  }
}

// Long segments: bitonic sort of (score desc, doc id asc, index asc) keys in
// shared memory (seg_len padded to a power of two, up to 16384 = 192 KB).
__device__ __forceinline__ uint32_t score_desc_key(float v) {
  uint32_t u = __float_as_uint(v == 0.f ? 0.f : v);          // -0 == +0
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);           // ascending in v
  return ~u;                                                 // descending in v
}

__global__ void topk_bitonic_kernel(const float* __restrict__ scores,
                                    const int32_t* __restrict__ ids, int seg_len, int n2, int k,
                                    int32_t* __restrict__ out_idx, float* __restrict__ out_score) {
  extern __shared__ uint8_t sm[];
  uint64_t* key = reinterpret_cast<uint64_t*>(sm);            // (score key << 32) | (id ^ sign)
  int32_t* pos = reinterpret_cast<int32_t*>(key + n2);
  const int seg = blockIdx.x;
  const float* sc = scores + (int64_t)seg * seg_len;
  const int32_t* id = ids + (int64_t)seg * seg_len;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    if (i < seg_len) {
      key[i] = ((uint64_t)score_desc_key(sc[i]) << 32) | (uint32_t)(id[i] ^ INT32_MIN);
      pos[i] = i;
    } else {
      key[i] = ~0ull;
      pos[i] = INT32_MAX;
    }
  }
  __syncthreads();
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (n2 >> 1); t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t a = key[lo], b = key[hi];
        const int32_t pa = pos[lo], pb = pos[hi];
        const bool gt = a > b || (a == b && pa > pb);
        if (gt == up) {
          key[lo] = b; key[hi] = a;
          pos[lo] = pb; pos[hi] = pa;
        }
      }
      __syncthreads();
    }
  }
  for (int r = threadIdx.x; r < k; r += blockDim.x) {
    const bool ok = r < seg_len;
    out_idx[(int64_t)seg * k + r] = ok ? pos[r] : -1;
    if (out_score) out_score[(int64_t)seg * k + r] = ok ? sc[pos[r]] : -CUDART_INF_F;
  }
}

// codec.py:82-95 / 98-115: code * scale[kvh][c]; INT4 low nibble first, sign-extended.
template <typename T>
__global__ void dequant_kernel(const uint8_t* __restrict__ codes, const float* __restrict__ scales,
                               int bits, int KVH, int D, int HD, T* __restrict__ out) {
  const int64_t total = (int64_t)KVH * D * HD;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int code;
    if (bits == 8) code = (int)(int8_t)codes[i];
    else {
      const uint8_t byte = codes[i >> 1];
      const int nib = (i & 1) ? (byte >> 4) : (byte & 0xF);
      code = (nib ^ 8) - 8;
    }
    const int h = (int)(i / ((int64_t)D * HD));
    const int c = (int)(i % HD);
    out[i] = Act<T>::from((float)code * scales[h * HD + c]);
  }
}

// codec.py:58-79 quantize_tensor, batched over n tensors [KVH][D][HD] (a whole
// pool page is 2L tensors).  Block = (tensor, kv head); thread i owns channels
// 2i, 2i+1.  scale = amax/level (1.0 for an all-zero channel), code =
// clamp(sign(y)*floor(|y|+0.5), +-level) with y = x/scale -- the reference's
// f32 operation order, so codes are bit-identical to the host codec.
// INT4 packs channel pairs low nibble first; each tensor is packed separately
// ((KVH*D*HD+1)/2 bytes), as in the HRKV payload.
template <typename T>
__global__ void quant_pages_kernel(const T* __restrict__ src, int D, int HD, int KVH, int bits,
                                   uint8_t* __restrict__ codes, float* __restrict__ scales) {
  const int t = blockIdx.x / KVH, h = blockIdx.x - t * KVH;
  const int c = 2 * threadIdx.x;
  if (c >= HD) return;
  const int64_t tensor_elems = (int64_t)KVH * D * HD;
  const T* x = src + t * tensor_elems + (int64_t)h * D * HD;
  float a0 = 0.f, a1 = 0.f;
  for (int d = 0; d < D; ++d) {
    a0 = fmaxf(a0, fabsf(Act<T>::to(x[(int64_t)d * HD + c])));
    a1 = fmaxf(a1, fabsf(Act<T>::to(x[(int64_t)d * HD + c + 1])));
  }
  const float level = bits == 8 ? 127.f : 7.f;
  const float s0 = a0 == 0.f ? 1.f : __fdiv_rn(a0, level);
  const float s1 = a1 == 0.f ? 1.f : __fdiv_rn(a1, level);
  float* so = scales + ((int64_t)t * KVH + h) * HD;
  so[c] = s0;
  so[c + 1] = s1;
  const int64_t tensor_bytes = bits == 8 ? tensor_elems : (tensor_elems + 1) / 2;
  uint8_t* co = codes + t * tensor_bytes;
  for (int d = 0; d < D; ++d) {
    const int64_t e = ((int64_t)h * D + d) * HD + c;
    const float y0 = __fdiv_rn(Act<T>::to(x[(int64_t)d * HD + c]), s0);
    const float y1 = __fdiv_rn(Act<T>::to(x[(int64_t)d * HD + c + 1]), s1);
    const float r0 = fminf(fmaxf(copysignf(floorf(__fadd_rn(fabsf(y0), 0.5f)), y0), -level), level);
    const float r1 = fminf(fmaxf(copysignf(floorf(__fadd_rn(fabsf(y1), 0.5f)), y1), -level), level);
    const int q0 = (int)r0, q1 = (int)r1;
    if (bits == 8) {
      co[e] = (uint8_t)(int8_t)q0;
      co[e + 1] = (uint8_t)(int8_t)q1;
    } else {
      co[e >> 1] = (uint8_t)((q0 & 0xF) | ((q1 & 0xF) << 4));   // e even: low nibble first
    }
  }
}

// codec.py:82-95 dequantize_tensor, batched over n tensors (whole page).
template <typename T>
__global__ void dequant_pages_kernel(const uint8_t* __restrict__ codes,
                                     const float* __restrict__ scales, int n, int bits, int KVH,
                                     int D, int HD, T* __restrict__ out) {
  const int64_t te = (int64_t)KVH * D * HD;
  const int64_t tb = bits == 8 ? te : (te + 1) / 2;
  const int64_t total = te * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / te, r = i - t * te;
    int code;
    if (bits == 8) code = (int)(int8_t)codes[t * tb + r];
    else {
      const uint8_t byte = codes[t * tb + (r >> 1)];
      code = (((r & 1) ? (byte >> 4) : (byte & 0xF)) ^ 8) - 8;
    }
    const int h = (int)(r / ((int64_t)D * HD));
    const int c = (int)(r % HD);
    out[i] = Act<T>::from((float)code * scales[(t * KVH + h) * HD + c]);
  }
}

// Vectorised form for the streaming path (host tier -> staging, once per
// document per step): one thread expands 16 consecutive codes of one row
// (16-byte / 8-byte code load, 16 channel scales, 32/64-byte store); grid.y
// walks (tensor, kv_head) so no 64-bit division per element.  Same per-element
// arithmetic as dequant_pages_kernel (f32 code*scale, then round to T).
template <typename T, int BITS>
__global__ void __launch_bounds__(256) dequant_pages_vec_kernel(
    const uint8_t* __restrict__ codes, const float* __restrict__ scales, int KVH, int D, int HD,
    T* __restrict__ out) {
  const int th = blockIdx.y;                    // t * KVH + h
  const int t = th / KVH, h = th - t * KVH;
  const int64_t te = (int64_t)KVH * D * HD;
  const int64_t tb = BITS == 8 ? te : te / 2;
  const int chunks = D * HD / 16;               // per (tensor, head)
  const int64_t head0 = (int64_t)h * D * HD;    // element offset of the head in its tensor
  const float* sc = scales + (int64_t)th * HD;
  T* o = out + t * te + head0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < chunks; j += gridDim.x * blockDim.x) {
    const int e = j * 16;
    const int c = e % HD;
    int q[16];
    if constexpr (BITS == 8) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(codes + t * tb + head0 + e));
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int i = 0; i < 16; ++i) q[i] = (int)(int8_t)(w[i >> 2] >> (8 * (i & 3)));
    } else {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(codes + t * tb + (head0 + e) / 2));
      const uint32_t w[2] = {v.x, v.y};
#pragma unroll
      for (int i = 0; i < 16; ++i) q[i] = (int)(((w[i >> 3] >> (4 * (i & 7))) & 0xF) ^ 8) - 8;
    }
    alignas(16) T r[16];
#pragma unroll
    for (int i = 0; i < 16; i += 4) {
      const float4 s4 = __ldg(reinterpret_cast<const float4*>(sc + c + i));
      r[i + 0] = Act<T>::from((float)q[i + 0] * s4.x);
      r[i + 1] = Act<T>::from((float)q[i + 1] * s4.y);
      r[i + 2] = Act<T>::from((float)q[i + 2] * s4.z);
      r[i + 3] = Act<T>::from((float)q[i + 3] * s4.w);
    }
    uint4* dst = reinterpret_cast<uint4*>(o + e);
    const uint4* srcv = reinterpret_cast<const uint4*>(r);
#pragma unroll
    for (int i = 0; i < (int)(16 * sizeof(T) / 16); ++i) dst[i] = srcv[i];
  }
}

static unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)device_sm_count() * 32;
  return (unsigned)std::max<int64_t>(1, std::min(g, cap));
}

static int do_gemm(int backend, int act, const void* A, const void* B, int64_t M, int N, int K,
                   const EpiParams& ep, cudaStream_t s) {
  if (backend == KRR_GEMM_AUTO) {
    // tensor cores for 16-bit operands whenever the tile constraints hold
    // (K % 64, N % 32, 16-byte aligned operands); CUDA-core kernel otherwise
    // (e.g. the reference's default desk config, d=128 with 16-wide heads, is
    // fine; odd widths are not)
    const bool glu = ep.kind == KRR_EPI_GLU_GELU || ep.kind == KRR_EPI_GLU_SILU;
    const bool tc_ok = act != KRR_F32 && K % 64 == 0 && N % (glu ? 64 : 32) == 0 &&
                       (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(B) & 15) == 0;
    backend = tc_ok ? KRR_GEMM_TCGEN05 : KRR_GEMM_SIMT;
  }
  ProfScope ps(s, 0, 2.0 * (double)M * N * K);
  if (backend == KRR_GEMM_TCGEN05) return launch_gemm_tcgen05(act, A, B, M, N, K, ep, s);
  return launch_gemm_simt(act, A, B, M, N, K, ep, s);
}

static int do_attention(int backend, int act, const AttnParams& p, cudaStream_t s) {
  if (backend == KRR_ATTN_AUTO) {
    const bool mma_hd = p.head_dim == 64 || p.head_dim == 128 || p.head_dim == 256;
    if (act == KRR_F32) backend = KRR_ATTN_SIMT;
    else if (attention_tcgen05_supported(act, p)) backend = KRR_ATTN_TCGEN05;
    else backend = mma_hd ? KRR_ATTN_MMA : KRR_ATTN_SIMT;   // any other head_dim
  }
  ProfScope ps(s, 1);
  if (p.prefix_bits != 0 && p.prefix_bits != 16) {
    // quantised prefix pages are expanded inside the TMEM-P kernel only
    if (backend != KRR_ATTN_TCGEN05 || p.head_dim > 128)
      return fail(KRR_EUNSUPPORTED, "quantised prefix pages need the tcgen05 attention with "
                                    "head_dim 64|128 and 16-bit activations");
    return launch_attention_fa(act, p, s);
  }
  if (backend == KRR_ATTN_TCGEN05) return launch_attention_fa(act, p, s);
  if (backend == KRR_ATTN_MMA) return launch_attention_mma(act, p, s);
  return launch_attention_simt(act, p, s);
}

template <typename T>
static void rmsnorm_launch(const float* x, const float* gain, int64_t rows, int d, T* out,
                           cudaStream_t s) {
  const int q = d / 4;
  if (d % 4 == 0 && q % 32 == 0) {
    int vpt = 1;
    while (q / vpt > 256 && vpt < 8) vpt *= 2;
    const int threads = q / vpt;
    if (threads * vpt == q && threads % 32 == 0 && threads <= 1024) {
      switch (vpt) {
        case 1: rmsnorm_vec_kernel<T, 1><<<(unsigned)rows, threads, 0, s>>>(x, gain, d, out); return;
        case 2: rmsnorm_vec_kernel<T, 2><<<(unsigned)rows, threads, 0, s>>>(x, gain, d, out); return;
        case 4: rmsnorm_vec_kernel<T, 4><<<(unsigned)rows, threads, 0, s>>>(x, gain, d, out); return;
        case 8: rmsnorm_vec_kernel<T, 8><<<(unsigned)rows, threads, 0, s>>>(x, gain, d, out); return;
      }
    }
  }
  rmsnorm_kernel<T><<<(unsigned)rows, d >= 1024 ? 256 : 128, 0, s>>>(x, gain, d, out);
}

static int do_rmsnorm(const float* x, const float* gain, int64_t rows, int d, int act, void* out,
                      cudaStream_t s) {
  ProfScope ps(s, 2);
  if (act == KRR_F32) rmsnorm_launch<float>(x, gain, rows, d, (float*)out, s);
  else if (act == KRR_F16) rmsnorm_launch<__half>(x, gain, rows, d, (__half*)out, s);
  else rmsnorm_launch<__nv_bfloat16>(x, gain, rows, d, (__nv_bfloat16*)out, s);
  return check_launch("rmsnorm");
}

}  // namespace krr

using namespace krr;

extern "C" {

const char* krr_last_error(void) { return g_err.c_str(); }
const char* krr_version(void) { return "kvrerank_b200 0.1 sm_100a"; }
uint64_t krr_launch_count(void) { return g_launches.load(); }

int krr_profile_enable(int enable) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = enable != 0;
  for (int i = 0; i < 3; ++i) { g_prof_ms[i] = 0; g_prof_n[i] = 0; }
  g_prof_flops = 0.0;
  for (auto& r : g_prof) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  g_prof.clear();
  return KRR_OK;
}

int krr_profile_read(double* ms_out3, uint64_t* n_out3, double* gemm_flops) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (auto& r : g_prof) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    g_prof_ms[r.cls] += ms;
    g_prof_n[r.cls] += 1;
    if (r.cls == 0) g_prof_flops += r.flops;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  for (int i = 0; i < 3; ++i) {
    if (ms_out3) ms_out3[i] = g_prof_ms[i];
    if (n_out3) n_out3[i] = g_prof_n[i];
  }
  if (gemm_flops) *gemm_flops = g_prof_flops;
  return KRR_OK;
}

int krr_init_uniform(uint64_t seed, double bound, int64_t rows, int64_t cols, int transpose,
                     int out_dtype, void* out, int64_t out_ld, krr_stream_t stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned g = grid_for(rows * cols, 256);
  if (out_dtype == KRR_F32)
    init_uniform_kernel<float><<<g, 256, 0, s>>>(seed, bound, rows, cols, transpose, (float*)out, out_ld);
  else if (out_dtype == KRR_F16)
    init_uniform_kernel<__half><<<g, 256, 0, s>>>(seed, bound, rows, cols, transpose, (__half*)out, out_ld);
  else
    init_uniform_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(seed, bound, rows, cols, transpose,
                                                         (__nv_bfloat16*)out, out_ld);
  return check_launch("init_uniform");
}

int krr_embed(const int32_t* tokens, const float* emb, int64_t rows, int32_t d, float* x,
              krr_stream_t stream) {
  return launch_embed(tokens, emb, rows, d, 1.0f, x, (cudaStream_t)stream);
}

int krr_rmsnorm(const float* x, const float* gain, int64_t rows, int32_t d, int out_dtype,
                void* out, krr_stream_t stream) {
  if (rows == 0) return KRR_OK;
  return do_rmsnorm(x, gain, rows, d, out_dtype, out, (cudaStream_t)stream);
}

int krr_gemm(int backend, int act_dtype, const void* A, const void* B, int64_t M, int32_t N,
             int32_t K, int epilogue, void* out, const krr_qkv_t* qkv, krr_stream_t stream) {
  EpiParams ep{};
  ep.kind = epilogue;
  ep.M = M;
  // gated epilogues write N/2 columns (act(gate) * up)
  ep.N = (epilogue == KRR_EPI_GLU_GELU || epilogue == KRR_EPI_GLU_SILU) ? N / 2 : N;
  ep.out = out;
  if (epilogue == KRR_EPI_QKV_ROPE) {
    KRR_REQUIRE(qkv != nullptr, KRR_ECONFIG, "QKV epilogue needs krr_qkv_t");
    ep.qkv = *qkv;
  }
  if (M == 0) return KRR_OK;
  return do_gemm(backend, act_dtype, A, B, M, N, K, ep, (cudaStream_t)stream);
}

int krr_attention(int backend, int act_dtype, const void* q, int32_t n_seqs, int32_t kv_heads,
                  int32_t group, int32_t head_dim, int32_t seq_len, int32_t prefix_len,
                  int32_t layer, int32_t cur_layer, void* const* prefix_kv,
                  const int32_t* prefix_valid_len, void* const* cur_kv,
                  const uint8_t* tok_valid, void* out, const void* prefix_pool,
                  int64_t prefix_pool_bytes, const void* cur_pool, int64_t cur_pool_bytes,
                  krr_stream_t stream) {
  return krr_attention_quant(backend, act_dtype, q, n_seqs, kv_heads, group, head_dim, seq_len,
                             prefix_len, layer, cur_layer, prefix_kv, prefix_valid_len, cur_kv,
                             tok_valid, out, prefix_pool, prefix_pool_bytes, cur_pool,
                             cur_pool_bytes, 16, nullptr, stream);
}

int krr_attention_quant(int backend, int act_dtype, const void* q, int32_t n_seqs,
                        int32_t kv_heads, int32_t group, int32_t head_dim, int32_t seq_len,
                        int32_t prefix_len, int32_t layer, int32_t cur_layer,
                        void* const* prefix_kv, const int32_t* prefix_valid_len,
                        void* const* cur_kv, const uint8_t* tok_valid, void* out,
                        const void* prefix_pool, int64_t prefix_pool_bytes, const void* cur_pool,
                        int64_t cur_pool_bytes, int32_t prefix_bits, const float* prefix_scales,
                        krr_stream_t stream) {
  AttnParams p{q, n_seqs, kv_heads, group, head_dim, seq_len, prefix_len, layer, cur_layer,
               prefix_kv, prefix_valid_len, cur_kv, tok_valid, out, prefix_pool,
               prefix_pool_bytes, cur_pool, cur_pool_bytes, prefix_bits, prefix_scales, nullptr,
               nullptr};
  if (n_seqs == 0) return KRR_OK;
  return do_attention(backend, act_dtype, p, (cudaStream_t)stream);
}

int krr_attention_occupancy(int act_dtype, int32_t head_dim, int32_t* ctas_per_sm) {
  KRR_REQUIRE(ctas_per_sm != nullptr, KRR_ECONFIG, "null argument");
  return attention_tcgen05_occupancy(act_dtype, head_dim, ctas_per_sm);
}

int krr_score_head(const float* x, int32_t n_seqs, int32_t seq_len, int32_t d,
                   const int32_t* last_index, const float* final_gain, const float* head,
                   float* scores, krr_stream_t stream) {
  if (n_seqs == 0) return KRR_OK;
  ProfScope ps((cudaStream_t)stream, 2);
  score_kernel<<<n_seqs, 256, 0, (cudaStream_t)stream>>>(x, seq_len, d, last_index, final_gain, head, scores);
  return check_launch("score_head");
}

int krr_segmented_topk(const float* scores, const int32_t* doc_ids, int32_t n_seg,
                       int32_t seg_len, int32_t k, int32_t* out_idx, float* out_score,
                       krr_stream_t stream) {
  KRR_REQUIRE(seg_len >= 0 && seg_len <= 16384, KRR_ESHAPE, "top-k segment too long");
  KRR_REQUIRE(k >= 1, KRR_ECONFIG, "top-k needs k >= 1");
  if (n_seg == 0) return KRR_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (seg_len <= 2048) {
    // rank by counting: O(n^2 / threads), 8 B of smem per candidate (<= 16 KB)
    const size_t smem = (size_t)seg_len * 8;
    topk_kernel<<<n_seg, 256, smem, s>>>(scores, doc_ids, seg_len, k, out_idx, out_score);
    return check_launch("segmented_topk");
  }
  int n2 = 1;
  while (n2 < seg_len) n2 <<= 1;
  const int smem = n2 * 12;                                  // <= 192 KB at 16384
  const int rc = ensure_func_smem((const void*)topk_bitonic_kernel, 16384 * 12);
  if (rc) return rc;
  topk_bitonic_kernel<<<n_seg, 1024, smem, s>>>(scores, doc_ids, seg_len, n2, k, out_idx,
                                                out_score);
  return check_launch("segmented_topk_bitonic");
}

int krr_dequant_kv(const uint8_t* codes, const float* scales, int32_t bits, int32_t kv_heads,
                   int32_t doc_len, int32_t head_dim, int out_dtype, void* out,
                   krr_stream_t stream) {
  KRR_REQUIRE(bits == 8 || bits == 4, KRR_ECONFIG, "dequant bits must be 8 or 4");
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned g = grid_for((int64_t)kv_heads * doc_len * head_dim, 256);
  if (out_dtype == KRR_F32)
    dequant_kernel<float><<<g, 256, 0, s>>>(codes, scales, bits, kv_heads, doc_len, head_dim, (float*)out);
  else if (out_dtype == KRR_F16)
    dequant_kernel<__half><<<g, 256, 0, s>>>(codes, scales, bits, kv_heads, doc_len, head_dim, (__half*)out);
  else
    dequant_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(codes, scales, bits, kv_heads, doc_len, head_dim,
                                                    (__nv_bfloat16*)out);
  return check_launch("dequant_kv");
}

int krr_quant_pages(const void* src, int src_dtype, int32_t n_tensors, int32_t kv_heads,
                    int32_t doc_len, int32_t head_dim, int32_t bits, uint8_t* codes,
                    float* scales, krr_stream_t stream) {
  KRR_REQUIRE(bits == 8 || bits == 4, KRR_ECONFIG, "quant bits must be 8 or 4");
  KRR_REQUIRE(head_dim % 2 == 0 && head_dim <= 2048, KRR_ESHAPE, "head_dim must be even");
  if (n_tensors == 0) return KRR_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned blocks = (unsigned)(n_tensors * kv_heads), threads = (unsigned)(head_dim / 2);
  if (src_dtype == KRR_F32)
    quant_pages_kernel<float><<<blocks, threads, 0, s>>>((const float*)src, doc_len, head_dim,
                                                          kv_heads, bits, codes, scales);
  else if (src_dtype == KRR_F16)
    quant_pages_kernel<__half><<<blocks, threads, 0, s>>>((const __half*)src, doc_len, head_dim,
                                                           kv_heads, bits, codes, scales);
  else
    quant_pages_kernel<__nv_bfloat16><<<blocks, threads, 0, s>>>(
        (const __nv_bfloat16*)src, doc_len, head_dim, kv_heads, bits, codes, scales);
  return check_launch("quant_pages");
}

int krr_dequant_pages(const uint8_t* codes, const float* scales, int32_t bits, int32_t n_tensors,
                      int32_t kv_heads, int32_t doc_len, int32_t head_dim, int out_dtype,
                      void* out, krr_stream_t stream) {
  KRR_REQUIRE(bits == 8 || bits == 4, KRR_ECONFIG, "dequant bits must be 8 or 4");
  if (n_tensors == 0) return KRR_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const bool vec = head_dim % 16 == 0 && (reinterpret_cast<uintptr_t>(codes) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(scales) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                   (int64_t)n_tensors * kv_heads <= 65535;
  if (vec) {
    const int chunks = doc_len * head_dim / 16;
    const dim3 grid((unsigned)std::max(1, std::min((chunks + 255) / 256, 64)),
                    (unsigned)(n_tensors * kv_heads));
#define KRR_DQ(T, B) \
  dequant_pages_vec_kernel<T, B><<<grid, 256, 0, s>>>(codes, scales, kv_heads, doc_len, head_dim, (T*)out)
    if (out_dtype == KRR_F32) { if (bits == 8) KRR_DQ(float, 8); else KRR_DQ(float, 4); }
    else if (out_dtype == KRR_F16) { if (bits == 8) KRR_DQ(__half, 8); else KRR_DQ(__half, 4); }
    else { if (bits == 8) KRR_DQ(__nv_bfloat16, 8); else KRR_DQ(__nv_bfloat16, 4); }
#undef KRR_DQ
    return check_launch("dequant_pages");
  }
  const unsigned g = grid_for((int64_t)n_tensors * kv_heads * doc_len * head_dim, 256);
  if (out_dtype == KRR_F32)
    dequant_pages_kernel<float><<<g, 256, 0, s>>>(codes, scales, n_tensors, bits, kv_heads,
                                                  doc_len, head_dim, (float*)out);
  else if (out_dtype == KRR_F16)
    dequant_pages_kernel<__half><<<g, 256, 0, s>>>(codes, scales, n_tensors, bits, kv_heads,
                                                   doc_len, head_dim, (__half*)out);
  else
    dequant_pages_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(codes, scales, n_tensors, bits,
                                                          kv_heads, doc_len, head_dim,
                                                          (__nv_bfloat16*)out);
  return check_launch("dequant_pages");
}

// ------------------------------------------------------------- layer loop
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Attention item-table entries for any split of `rows` into sequences (n <= rows,
// n * Rp <= (G + 63) * rows): the grouped-attention table lives in the workspace.
static int64_t items_bound(const krr_model_t* m, int64_t rows) {
  const int64_t G = m->heads / (m->kv_heads > 0 ? m->kv_heads : 1);
  const int64_t ir = attention_item_rows(m->head_dim);
  return (int64_t)m->kv_heads * (((G + 63) * rows + ir - 1) / ir + rows);
}

int krr_workspace_bytes(const krr_model_t* m, int64_t rows, size_t* out) {
  KRR_REQUIRE(m && out, KRR_ECONFIG, "null argument");
  const size_t es = dtype_size(m->act_dtype);
  const int64_t d = m->model_dim, hq = (int64_t)m->heads * m->head_dim;
  size_t total = align256(rows * d * 4)          // x  (f32 residual stream)
               + align256(rows * d * es)         // xn (normed activations)
               + align256(rows * hq * es)        // q  ([unit][g*t][hd])
               + align256(rows * hq * es)        // attention output
               + align256(rows * (int64_t)ffn_of(m) * es)     // MLP hidden
               + align256(16 * items_bound(m, rows) + 16);    // attention item table
  *out = total;
  return KRR_OK;
}

int krr_forward(const krr_model_t* m, const krr_batch_t* b, void* workspace, size_t ws_bytes,
                krr_stream_t stream) {
  KRR_REQUIRE(m && b, KRR_ECONFIG, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  const int L = m->layers, d = m->model_dim, H = m->heads, KVH = m->kv_heads, HD = m->head_dim;
  KRR_REQUIRE(H % KVH == 0 && H * HD == d, KRR_ECONFIG, "inconsistent model geometry");
  KRR_REQUIRE(m->mlp_kind >= KRR_MLP_GELU && m->mlp_kind <= KRR_MLP_SWIGLU, KRR_ECONFIG,
              "unknown mlp_kind");
  const int G = H / KVH;
  const int F = ffn_of(m);
  const bool gated = m->mlp_kind != KRR_MLP_GELU;
  KRR_REQUIRE(!gated || F % 32 == 0, KRR_ECONFIG, "gated MLP needs ffn_dim % 32 == 0");
  const int n_up = gated ? 2 * F : F;                 // up-projection GEMM width
  const int64_t rows = (int64_t)b->n_seqs * b->seq_len;
  if (rows == 0) return KRR_OK;
  KRR_REQUIRE(b->positions || b->pos0 + b->seq_len <= m->max_position, KRR_ESHAPE,
              "positions exceed max_position");
  KRR_REQUIRE(b->cur_kv_layers == 1 || b->cur_kv_layers == L, KRR_ECONFIG,
              "cur_kv_layers must be 1 or layers");
  size_t need = 0;
  krr_workspace_bytes(m, rows, &need);
  KRR_REQUIRE(ws_bytes >= need, KRR_ECONFIG, "workspace too small");
  const int act = m->act_dtype;
  const size_t es = dtype_size(act);
  uint8_t* w = static_cast<uint8_t*>(workspace);
  float* x = reinterpret_cast<float*>(w);          w += align256(rows * d * 4);
  void* xn = w;                                    w += align256(rows * d * es);
  void* qb = w;                                    w += align256(rows * (int64_t)H * HD * es);
  void* ab = w;                                    w += align256(rows * (int64_t)H * HD * es);
  void* hb = w;                                    w += align256(rows * (int64_t)ffn_of(m) * es);
  int* item_count = reinterpret_cast<int*>(w);
  void* items = w + 16;

  int rc = KRR_OK;
  if (b->x_in) {
    if (cudaMemcpyAsync(x, b->x_in, rows * d * sizeof(float), cudaMemcpyDeviceToDevice, s) !=
        cudaSuccess)
      return fail(KRR_ECUDA, "x_in copy failed");
  } else {
    rc = launch_embed(b->tokens, m->token_embedding, rows, d,
                      m->embed_scale > 0.f ? m->embed_scale : 1.0f, x, s);
    if (rc) return rc;
  }
  // cached-prefix scoring: group sequences that share a document so attention
  // streams each document's K/V once per 256 rows of all its queries
  const bool grouped = b->prefix_len > 0 && act != KRR_F32 &&
                       (HD == 64 || HD == 128 || HD == 256);
  const int item_rows = attention_item_rows(HD);
  if (grouped) {
    rc = build_attention_items(b->prefix_kv, b->n_seqs, G, b->seq_len, KVH, item_rows, items,
                               items_bound(m, rows), item_count, s);
    if (rc) return rc;
  }
  const int nqkv = (H + 2 * KVH) * HD;
  const bool prefill_only = b->scores == nullptr && b->x_out == nullptr;
  // last-layer row pruning needs the compact buffers to fit the dead regions
  const bool scoring_tail = b->scores != nullptr && b->x_out == nullptr &&
                            b->last_index != nullptr && b->seq_len >= 4 &&
                            (int64_t)b->seq_len * H * HD >= F;
  for (int l = 0; l < L; ++l) {
    rc = do_rmsnorm(x, m->attn_gain[l], rows, d, act, xn, s);
    if (rc) return rc;
    EpiParams ep{};
    ep.kind = KRR_EPI_QKV_ROPE;
    ep.M = rows;
    ep.N = nqkv;
    const int cl = b->cur_kv_layers == 1 ? 0 : l;
    ep.qkv = krr_qkv_t{H, KVH, HD, b->seq_len, b->pos0, cl, b->seq_len,
                       m->rope_cos, m->rope_sin, qb, b->cur_kv, b->positions};
    rc = do_gemm(m->gemm_backend, act, xn, m->wqkv[l], rows, nqkv, d, ep, s);
    if (rc) return rc;
    // Prefill needs only K/V from the last layer: the rest of that layer
    // cannot influence any stored byte (model.py:365-400 dataflow).
    if (prefill_only && l == L - 1) break;
    AttnParams ap{qb, b->n_seqs, KVH, G, HD, b->seq_len, b->prefix_len, l, cl,
                  b->prefix_kv, b->prefix_valid_len, b->cur_kv, b->tok_valid, ab,
                  b->prefix_pool, b->prefix_pool_bytes, b->cur_pool, b->cur_pool_bytes,
                  b->prefix_bits, b->prefix_scales, grouped ? items : nullptr,
                  grouped ? item_count : nullptr, item_rows};
    rc = do_attention(m->attn_backend, act, ap, s);
    if (rc) return rc;
    EpiParams er{};
    er.kind = KRR_EPI_RESIDUAL;
    er.out = x;
    EpiParams eg{};
    eg.kind = !gated ? KRR_EPI_GELU
              : m->mlp_kind == KRR_MLP_GEGLU ? KRR_EPI_GLU_GELU : KRR_EPI_GLU_SILU;
    eg.N = F;   // output width (the hidden); the GEMM itself is n_up wide
    if (scoring_tail && l == L - 1) {
      // Only the scored row of each sequence reaches the score head
      // (reranker.py:211-212): run this layer's WO + MLP on n rows.  Compact
      // buffers reuse regions that are dead by now (q, xn, hb, ab).
      const int64_t n = b->n_seqs;
      void* ab_c = qb;                                      // [n, H*HD] act
      float* x_c = reinterpret_cast<float*>(xn);            // [n, d] f32
      void* xn_c = hb;                                      // [n, d] act
      void* hb_c = ab;                                      // [n, F] act
      {
        ProfScope ps(s, 2);
        if (es == 2)
          gather_last_kernel<uint16_t><<<(unsigned)n, 256, 0, s>>>((const uint16_t*)ab, b->last_index, b->seq_len, H * HD, (uint16_t*)ab_c);
        else
          gather_last_kernel<float><<<(unsigned)n, 256, 0, s>>>((const float*)ab, b->last_index, b->seq_len, H * HD, (float*)ab_c);
        gather_last_kernel<float><<<(unsigned)n, 256, 0, s>>>((const float*)x, b->last_index, b->seq_len, d, x_c);
        rc = check_launch("gather_last");
        if (rc) return rc;
      }
      er.M = n; er.N = d; er.out = x_c;
      rc = do_gemm(m->gemm_backend, act, ab_c, m->wo[l], n, d, H * HD, er, s);
      if (rc) return rc;
      rc = do_rmsnorm(x_c, m->mlp_gain[l], n, d, act, xn_c, s);
      if (rc) return rc;
      eg.M = n; eg.out = hb_c;
      rc = do_gemm(m->gemm_backend, act, xn_c, m->w_up[l], n, n_up, d, eg, s);
      if (rc) return rc;
      rc = do_gemm(m->gemm_backend, act, hb_c, m->w_down[l], n, d, F, er, s);
      if (rc) return rc;
      return krr_score_head(x_c, b->n_seqs, 1, d, nullptr, m->final_gain, m->score_head,
                            b->scores, stream);
    }
    er.M = rows;
    er.N = d;
    rc = do_gemm(m->gemm_backend, act, ab, m->wo[l], rows, d, H * HD, er, s);
    if (rc) return rc;
    rc = do_rmsnorm(x, m->mlp_gain[l], rows, d, act, xn, s);
    if (rc) return rc;
    eg.M = rows;
    eg.out = hb;
    rc = do_gemm(m->gemm_backend, act, xn, m->w_up[l], rows, n_up, d, eg, s);
    if (rc) return rc;
    rc = do_gemm(m->gemm_backend, act, hb, m->w_down[l], rows, d, F, er, s);
    if (rc) return rc;
  }
  if (b->x_out &&
      cudaMemcpyAsync(b->x_out, x, rows * d * sizeof(float), cudaMemcpyDeviceToDevice, s) !=
          cudaSuccess)
    return fail(KRR_ECUDA, "x_out copy failed");
  if (b->scores) {
    KRR_REQUIRE(b->last_index != nullptr, KRR_ECONFIG, "scores need last_index");
    rc = krr_score_head(x, b->n_seqs, b->seq_len, d, b->last_index, m->final_gain,
                        m->score_head, b->scores, stream);
    if (rc) return rc;
  }
  return KRR_OK;
}

}  // extern "C"
