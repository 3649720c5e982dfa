// Internal launcher declarations shared across the .cu files.
#pragma once
#include "common.cuh"

namespace krr {

// Epilogue parameters shared by the tcgen05 and SIMT GEMMs.
struct EpiParams {
  int kind;      // KRR_EPI_*
  int64_t M;
  int N;
  void* out;     // STORE/GELU: act [M,N]; RESIDUAL: f32 [M,N]
  krr_qkv_t qkv; // QKV_ROPE scatter
};

int launch_gemm_tcgen05(int act_dtype, const void* A, const void* B, int64_t M, int N, int K,
                        const EpiParams& ep, cudaStream_t s);
int launch_gemm_simt(int act_dtype, const void* A, const void* B, int64_t M, int N, int K,
                     const EpiParams& ep, cudaStream_t s);

struct AttnParams {
  const void* q;               // [units][group*seq_len][hd]
  int n_seqs, kv_heads, group, head_dim, seq_len, prefix_len, layer, cur_layer;
  void* const* prefix_kv;
  const int32_t* prefix_valid_len;
  void* const* cur_kv;
  const uint8_t* tok_valid;
  void* out;                   // [n_seqs*seq_len][heads*hd]
  // base/extent of the allocations the prefix_kv / cur_kv pointers point into
  // (the tcgen05 kernel addresses them as TMA pages); may be null
  const void* prefix_pool;
  int64_t prefix_pool_bytes;
  const void* cur_pool;
  int64_t cur_pool_bytes;
  // prefix page element: 16-bit (0 or 16), or HRKV INT8 / INT4 codes (8 / 4)
  // with per-(page, channel) f32 scales [page][head_dim]; pages then hold
  // prefix_len * head_dim * bits / 8 bytes and prefix_pool is the code pool
  int prefix_bits;
  const float* prefix_scales;
  // grouped work items from build_attention_items (sequences sharing a prefix
  // document, adjacent in the batch, attend as one row group); null = per seq
  const void* items;
  const int* n_items;
  int item_rows;               // rows per item the table was built for
};
// query rows per attention work item (256: two 128-row tiles; 128 at head_dim 256)
int attention_item_rows(int head_dim);
int64_t attention_items_capacity(int64_t n_seqs, int group, int seq_len, int kv_heads,
                                 int item_rows);
int build_attention_items(void* const* prefix_kv, int n_seqs, int group, int seq_len,
                          int kv_heads, int item_rows, void* items, int64_t cap, int* count,
                          cudaStream_t s);
int launch_attention_mma(int act_dtype, const AttnParams& p, cudaStream_t s);
int launch_attention_fa(int act_dtype, const AttnParams& p, cudaStream_t s);
bool attention_tcgen05_supported(int act_dtype, const AttnParams& p);
int attention_tcgen05_occupancy(int act_dtype, int head_dim, int* out);
int launch_attention_simt(int act_dtype, const AttnParams& p, cudaStream_t s);

int device_sm_count();

}  // namespace krr
