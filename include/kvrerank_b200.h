/*
 * kvrerank_b200.h — C ABI of the B200-native KV-reuse rerank hot path.
 *
 * One shared library (paper_2504_02921_b200/_kvrerank_b200.so) exports these
 * entry points.  Signatures use plain pointers, sizes and cudaStream_t only
 * (no torch types).  Every call is asynchronous on the given stream, returns
 * 0 on success or a KRR_E* code, and leaves a message for krr_last_error()
 * (thread-local).  Device buffers are owned by the caller; the library keeps
 * only a cache of TMA descriptors keyed by pointer/shape.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/kvrerank/):
 *   krr_init_uniform      <- model.py:123-129 _tensor + hashing.py:58-80 uniform_signed
 *   krr_forward           <- model.py:332-403 forward (the layer loop), as called by
 *                            reranker.py:182-201 doc_prefill (prefix_len == 0) and
 *                            reranker.py:204-212 _query_block (prefix = cached DocKV),
 *                            batched over many sequences in one M dimension
 *   krr_embed             <- model.py:352   x = token_embedding[tokens]
 *   krr_rmsnorm           <- model.py:439-441 _norm_rows
 *   krr_gemm              <- model.py:368,397,400 x@wqkv (+RoPE :370-371), attn@wo (+residual),
 *                            gelu(xn@w_up) (:444-446), @w_down (+residual)
 *   krr_attention         <- model.py:373-394 (+ _exp_rows :406-436)
 *   krr_attention_quant   <- the same over HRKV INT8/INT4 prefix pages, codec.py:82-95
 *                            dequantize_tensor fused in (pipeline.py:251-271 fetch+decode)
 *   krr_score_head        <- model.py:402 final norm + reranker.py:211-212 last-row dot
 *   krr_segmented_topk    <- pipeline.py:285-287 _select
 *   krr_dequant_kv        <- codec.py:82-95 dequantize_tensor (INT8/INT4 -> 16-bit pool page)
 *   krr_quant_pages       <- codec.py:58-79 quantize_tensor, batched over a page's 2L tensors
 *   krr_dequant_pages     <- codec.py:82-95 dequantize_tensor, batched (host-tier INT8/INT4)
 */
#ifndef KVRERANK_B200_H
#define KVRERANK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* krr_stream_t; /* == cudaStream_t */

/* status codes (mapped to the reference's errors.py classes by the host layer) */
enum {
  KRR_OK = 0,
  KRR_ECONFIG = 1,   /* -> ConfigError   */
  KRR_ESHAPE = 2,    /* -> ShapeError    */
  KRR_ECUDA = 3,     /* -> RuntimeError (CUDA failure)   */
  KRR_EUNSUPPORTED = 4
};

/* element types */
enum { KRR_F32 = 0, KRR_F16 = 1, KRR_BF16 = 2 };

/* GEMM epilogues: C = A[M,K] . B[N,K]^T  (both K-major) */
enum {
  KRR_EPI_STORE = 0,     /* out[M,N] (act dtype) = C                         */
  KRR_EPI_GELU = 1,      /* out[M,N] (act dtype) = gelu_tanh(C)              */
  KRR_EPI_RESIDUAL = 2,  /* resid[M,N] (f32) += C                            */
  KRR_EPI_QKV_ROPE = 3,  /* RoPE(q,k) then scatter q / k / v (see krr_qkv_t)  */
  /* gated MLP (architecture variants): B's rows interleave
   * 32-row blocks of the gate and up projections (block 2p = gate rows
   * 32p..32p+31, block 2p+1 = up rows 32p..32p+31); N % 64 == 0 and
   * out[M, N/2] (act dtype) = act(gate) * up                               */
  KRR_EPI_GLU_GELU = 4,  /* GeGLU  (Gemma): gelu_tanh(gate) * up             */
  KRR_EPI_GLU_SILU = 5   /* SwiGLU (Mistral/Llama): silu(gate) * up         */
};

/* MLP kinds (krr_model_t.mlp_kind) */
enum { KRR_MLP_GELU = 0 /* reference: gelu_tanh(x W_up) W_down, 4d */,
       KRR_MLP_GEGLU = 1, KRR_MLP_SWIGLU = 2 };

/* GEMM backends */
enum { KRR_GEMM_AUTO = 0, KRR_GEMM_TCGEN05 = 1, KRR_GEMM_SIMT = 2 };

/* attention backends: auto picks TCGEN05 when the pools are described and the
 * geometry is supported (16-bit, head_dim 64/128/256), else MMA (16-bit) / SIMT (f32) */
enum { KRR_ATTN_AUTO = 0, KRR_ATTN_MMA = 1, KRR_ATTN_SIMT = 2, KRR_ATTN_TCGEN05 = 3 };

/* Scatter description for KRR_EPI_QKV_ROPE.  Row r of the GEMM is token
 * t = r % seq_len of sequence b = r / seq_len at absolute position pos0 + t.
 * q  -> q_out[b][kvh][g][t][hd]           (GQA rows packed, model.py:377-378)
 * k,v-> kv_seq[b] + ((layer*2 + {0,1})*kv_heads + kvh)*kv_len*hd + t*hd + c  */
typedef struct {
  int32_t heads, kv_heads, head_dim, seq_len, pos0, layer, kv_len;
  const float* rope_cos;   /* [max_position, hd/2] */
  const float* rope_sin;
  void* q_out;
  void* const* kv_seq;     /* device array [n_seqs] of KV slab pointers */
  /* device [n_seqs*seq_len] absolute RoPE positions (model.py:358 takes any
   * strictly increasing positions), or NULL: row r sits at pos0 + r % seq_len */
  const int32_t* positions;
} krr_qkv_t;

/* Model: per-layer weights are K-major ([out, in]) in act dtype (f32/f16/bf16). */
typedef struct {
  int32_t layers, model_dim, heads, kv_heads, head_dim, vocab_size, max_position;
  int32_t act_dtype;              /* KRR_F32 (debug), KRR_F16 or KRR_BF16 */
  int32_t gemm_backend;           /* KRR_GEMM_* */
  int32_t attn_backend;           /* KRR_ATTN_* */
  const float* token_embedding;   /* [V, d] f32 */
  const float* rope_cos;          /* [max_position, hd/2] f32 */
  const float* rope_sin;
  const float* final_gain;        /* [d] */
  const float* score_head;        /* [d] */
  const float* const* attn_gain;  /* host array [L] of device [d] */
  const float* const* mlp_gain;
  const void* const* wqkv;        /* host array [L] of device [(H+2KVH)*HD, d] */
  const void* const* wo;          /* [d, H*HD] */
  const void* const* w_up;        /* [F, d] (gated kinds: [2F, d], gate/up 32-row interleave) */
  const void* const* w_down;      /* [d, F]   */
  /* architecture variants (zero-initialised = the reference model) */
  int32_t ffn_dim;                /* F; 0 = 4d                                  */
  int32_t mlp_kind;               /* KRR_MLP_*                                  */
  float embed_scale;              /* x = E[tok] * scale (Gemma: sqrt(d)); 0 = 1 */
} krr_model_t;

/* A batch of sequences run through the layer stack together.  Every
 * sequence has seq_len tokens at positions pos0..pos0+seq_len-1 on top of a
 * prefix of prefix_len cached positions. */
typedef struct {
  int32_t n_seqs, seq_len, pos0, prefix_len;
  int32_t cur_kv_layers;           /* layers held by each cur_kv slab: L (prefill into the
                                      pool) or 1 (per-layer suffix scratch, reused) */
  const int32_t* tokens;           /* device [n_seqs*seq_len] */
  const uint8_t* tok_valid;        /* device [n_seqs*seq_len] 1 = real token */
  const int32_t* prefix_valid_len; /* device [n_seqs] (ignored when prefix_len == 0) */
  void* const* prefix_kv;          /* device [n_seqs] KV slab ptrs [L][2][KVH][prefix_len][HD] */
  void* const* cur_kv;             /* device [n_seqs] KV slab ptrs [cur_kv_layers][2][KVH][seq_len][HD] */
  const int32_t* last_index;       /* device [n_seqs] row scored, or NULL */
  float* scores;                   /* device [n_seqs] out, or NULL */
  /* the allocations prefix_kv[] / cur_kv[] point into (pool slab, suffix
   * scratch): base + size in bytes; lets the tcgen05 attention address KV
   * pages through one TMA descriptor.  NULL/0 = unknown (slower kernel). */
  const void* prefix_pool;
  int64_t prefix_pool_bytes;
  const void* cur_pool;
  int64_t cur_pool_bytes;
  /* layer-split execution (teacher-forced checks, pipelined stacks): when
   * x_in is set the residual stream starts from it ([n_seqs*seq_len, d] f32)
   * instead of the embedding; when x_out is set the residual after the last
   * layer (before the final norm) is copied there and every layer runs in full. */
  const float* x_in;
  float* x_out;
  /* device [n_seqs*seq_len] absolute positions (RoPE), or NULL = pos0 + t;
   * the caller checks them against max_position */
  const int32_t* positions;
  /* prefix page format: 0/16 = act-dtype pages; 8 / 4 = HRKV INT8 / INT4 code
   * pages (codec.py:58-115; slot layout [L][2][KVH][prefix_len][head_dim] codes,
   * INT4 low nibble first) with f32 scales [page][head_dim] at prefix_scales,
   * page = (slot*L + layer)*2*KVH + {K,V}*KVH + kvh, dequantised inside the
   * attention kernel (head_dim 64|128, 16-bit activations) */
  int32_t prefix_bits;
  const float* prefix_scales;
} krr_batch_t;

const char* krr_last_error(void);
const char* krr_version(void);
uint64_t krr_launch_count(void);          /* kernels launched by this library so far */

/* Bytes of scratch krr_forward needs for n_seqs*seq_len rows. */
int krr_workspace_bytes(const krr_model_t* m, int64_t rows, size_t* out_bytes);

/* Full layer stack over a batch (embedding -> L layers -> final norm/score).
 * Replaces kvrerank/model.py:332-403 `forward` as called per pair by
 * reranker.py:182-201 (`doc_prefill`, prefix_len = 0: K/V written into pool
 * pages) and :204-212 (`_query_block`, prefix_len = D: suffix scoring), batched
 * over all pairs in one M dimension. */
int krr_forward(const krr_model_t* m, const krr_batch_t* b, void* workspace,
                size_t workspace_bytes, krr_stream_t stream);

/* Per-kernel timing of krr_forward (CUDA events on the launch stream).
 * enable!=0 turns recording on; krr_profile_read returns accumulated ms and
 * launch counts per kernel class: 0 gemm, 1 attention, 2 norm/embed/score. */
int krr_profile_enable(int enable);
int krr_profile_read(double* ms_out3, uint64_t* launches_out3, double* gemm_flops_out);

/* model.py:123-129 `_tensor` / hashing.py:58-80 `uniform_signed`: one named
 * SplitMix64 stream, written K-major ([out, in]) when transpose != 0. */
int krr_init_uniform(uint64_t stream_seed, double bound, int64_t rows, int64_t cols,
                     int transpose, int out_dtype, void* out, int64_t out_ld,
                     krr_stream_t stream);
/* model.py:352 token-embedding gather (f32 residual stream). */
int krr_embed(const int32_t* tokens, const float* emb, int64_t rows, int32_t d,
              float* x, krr_stream_t stream);
/* model.py:439-441 `_norm_rows` (x / sqrt(mean x^2 + eps) * gain). */
int krr_rmsnorm(const float* x, const float* gain, int64_t rows, int32_t d, int out_dtype,
                void* out, krr_stream_t stream);
/* model.py:368 (x @ wqkv + RoPE :370-371 + GQA pack :377-378), :397 (attn @ wo
 * + residual), :399-400 (gelu(xn @ w_up) @ w_down + residual); epilogue per KRR_EPI_*. */
int krr_gemm(int backend, int act_dtype, const void* A, const void* B, int64_t M, int32_t N,
             int32_t K, int epilogue, void* out, const krr_qkv_t* qkv, krr_stream_t stream);
/* model.py:373-394 attention over cached prefix K/V + causal suffix, with
 * `_exp_rows` :406-436 (shared max, masked rows -> 0, no 1/sqrt(HD)). */
int krr_attention(int backend, int act_dtype, const void* q, int32_t n_seqs, int32_t kv_heads,
                  int32_t group, int32_t head_dim, int32_t seq_len, int32_t prefix_len,
                  int32_t layer, int32_t cur_layer, void* const* prefix_kv,
                  const int32_t* prefix_valid_len, void* const* cur_kv,
                  const uint8_t* tok_valid, void* out, const void* prefix_pool,
                  int64_t prefix_pool_bytes, const void* cur_pool, int64_t cur_pool_bytes,
                  krr_stream_t stream);
/* krr_attention over quantised prefix pages (prefix_bits 8|4, see krr_batch_t):
 * codec.py:82-95 dequantize_tensor fused into model.py:373-394 -- the codes are
 * expanded to f16(code*scale) in shared memory, never written back to HBM. */
int krr_attention_quant(int backend, int act_dtype, const void* q, int32_t n_seqs,
                        int32_t kv_heads, int32_t group, int32_t head_dim, int32_t seq_len,
                        int32_t prefix_len, int32_t layer, int32_t cur_layer,
                        void* const* prefix_kv, const int32_t* prefix_valid_len,
                        void* const* cur_kv, const uint8_t* tok_valid, void* out,
                        const void* prefix_pool, int64_t prefix_pool_bytes, const void* cur_pool,
                        int64_t cur_pool_bytes, int32_t prefix_bits, const float* prefix_scales,
                        krr_stream_t stream);
/* Co-resident CTAs per SM of the tcgen05 attention kernel (diagnostic). */
int krr_attention_occupancy(int act_dtype, int32_t head_dim, int32_t* ctas_per_sm);
/* model.py:402 final norm + reranker.py:211-212 score of the last valid row
 * (the reference's d-vector head, or the yes/no lm_head-row difference). */
int krr_score_head(const float* x, int32_t n_seqs, int32_t seq_len, int32_t d,
                   const int32_t* last_index, const float* final_gain, const float* head,
                   float* scores, krr_stream_t stream);
/* pipeline.py:285-287 `_select`: top-k per segment by (score desc, doc_id asc).  scores/doc_ids [n_seg*seg_len];
 * out_idx [n_seg*k] (index within segment, -1 when k > seg_len). */
int krr_segmented_topk(const float* scores, const int32_t* doc_ids, int32_t n_seg,
                       int32_t seg_len, int32_t k, int32_t* out_idx, float* out_score,
                       krr_stream_t stream);
/* HRKV INT8/INT4 (codec.py:58-115) payload tensor [KVH][D][HD] -> 16-bit/f32 page. */
int krr_dequant_kv(const uint8_t* codes, const float* scales, int32_t bits, int32_t kv_heads,
                   int32_t doc_len, int32_t head_dim, int out_dtype, void* out,
                   krr_stream_t stream);

/* Batched HRKV quantisation of n tensors [KVH][D][HD] (e.g. one pool page = 2L
 * tensors): scales [n][KVH][HD] f32; codes per tensor KVH*D*HD bytes (INT8) or
 * (KVH*D*HD+1)/2 bytes (INT4, low nibble first).  Bit-identical to the host codec. */
int krr_quant_pages(const void* src, int src_dtype, int32_t n_tensors, int32_t kv_heads,
                    int32_t doc_len, int32_t head_dim, int32_t bits, uint8_t* codes,
                    float* scales, krr_stream_t stream);
int krr_dequant_pages(const uint8_t* codes, const float* scales, int32_t bits, int32_t n_tensors,
                      int32_t kv_heads, int32_t doc_len, int32_t head_dim, int out_dtype,
                      void* out, krr_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* KVRERANK_B200_H */
