// Shared declarations of the fused attention kernels.
#pragma once
#include "common.cuh"

namespace sc {

struct AttnArgs {
  const void* q;
  const void* k;
  const void* v;
  int64_t ld;
  void* out;
  int64_t ld_out;
  const int32_t* cu;
  const int32_t* qlen;
  int nseq, T, H, d;
  Links links;
  int padding;
  float scale;
  const uint8_t* flags;
  const int32_t* glob_cu;
  const int32_t* glob_pos;
  int32_t* status;
  int row_begin, row_end;  // token-row range to process (all-rows mode)
  // Head-row mode (generic kernel after the band kernel): items enumerate the
  // cls + query-group rows of every sequence through head_base; a FULL doc
  // link is served by merging the band kernel's per-tile partials.
  const int32_t* head_base;  // [nseq+1] or nullptr for all-rows mode
  int n_head_rows;
  const float* partials;     // [tiles*rec_per_tile][H][fmax][d+2]: (m, l, acc[d]); nullptr = scan doc keys
  const int32_t* tile_base;  // [nseq+1]
  int fmax;
  int rec_per_tile;          // partial records per doc tile (one per 16-row warp block)
};

bool load_links(const int32_t* links, Links* L);

// Tiled doc-band attention backward (attn_bwd_band.cu): bf16, head_dim 64, doc tiles of 64 rows.
struct BandBwdArgs {
  const __nv_bfloat16 *q, *k, *v, *out, *dout;
  int64_t ld, ld_out, ld_dout;
  void *dq, *dk, *dv;             // fp32, or bf16 when grad_bf16
  int grad_bf16;
  int64_t ld_grad;
  float2* stats;                  // [T*H] (lse, D), shared with the generic kernels
  const int32_t *cu, *qlen, *tile_base;
  int nseq, H, w;                 // w = doc->doc window
  Links links;
  int padding;
  float inv_scale;
  float* head_part;               // [tiles][H][2][NH][64] per-tile head-key dV / dK partials, or nullptr
  // head-row pass split over key ranges (head_ks > 1): per (seq, head, split) (m, l) and dQ partials
  float* head_split;              // [nseq][H][head_ks][NH][2 + 64]
  int head_ks, head_phase;
  int head_warps;                 // warps per head-row CTA (8, or 2 for short sequences)
};
// Gradient stores in fp32 or bf16 (element index idx of the buffer).
__device__ __forceinline__ void store_grad(void* base, int64_t idx, float v, int bf16) {
  if (bf16) reinterpret_cast<__nv_bfloat16*>(base)[idx] = __float2bfloat16_rn(v);
  else reinterpret_cast<float*>(base)[idx] = v;
}
__device__ __forceinline__ void store_grad2(void* base, int64_t idx, float a, float b, int bf16) {  // idx even
  if (bf16) *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(base) + idx) = __floats2bfloat162_rn(a, b);
  else *reinterpret_cast<float2*>(reinterpret_cast<float*>(base) + idx) = make_float2(a, b);
}
__device__ __forceinline__ void add_grad(void* base, int64_t idx, float v, int bf16) {
  if (bf16) {
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(base) + idx;
    *p = __float2bfloat16_rn(__bfloat162float(*p) + v);
  } else {
    reinterpret_cast<float*>(base)[idx] += v;
  }
}
// phase 0: doc-row statistics + dQ (+ head-key partials); 1: doc-key dK / dV; 2: head-key partial
// reduction; 3: head-row statistics + dQ.  max_head = 1 + max qgroup_len (<= 32); NH = 16 when max_head <= 16, else 32.
int launch_attn_bwd_band(const BandBwdArgs& a, int ntiles, int max_head, int phase, cudaStream_t st);
int launch_attn_generic(const AttnArgs& a, int dtype, cudaStream_t st);

// Rows of the query group that attend the whole document (FULL doc link):
// their split-softmax partials are produced per doc tile by the band kernel.
__host__ __device__ inline int full_rows_needed(const Links& L, int max_qgroup_len) {
  if (L.w[1][2] == SC_LINK_FULL) return 1 + max_qgroup_len;
  if (L.w[0][2] == SC_LINK_FULL) return 1;
  return 0;
}

// Tiled band kernel (attn_band_mma.cu).  Returns SC_ERR_UNSUPPORTED when the
// pattern/shape is outside its envelope (the caller then uses the generic kernel).
size_t band_workspace_bytes(int nseq, int T, int H, int d, int tile_rows, int max_qgroup_len,
                            const Links& L);
// doc_rows = false: head rows only (cls/query rows + CLS split-softmax records),
// used after the tcgen05 kernel has computed the doc rows.
int launch_attn_band(const AttnArgs& a, int dtype, const int32_t* seq_tile_base,
                     const int32_t* seq_head_base, int tile_rows, int max_qgroup_len, void* ws,
                     size_t ws_bytes, cudaStream_t st, bool doc_rows = true);

// merge_full_rows_kernel alone: folds the per-tile split-softmax records (band-kernel layout,
// 64-row tiles) into the head rows with a FULL doc link (used after the tcgen05 kernel).
int launch_head_merge(const AttnArgs& a, const int32_t* seq_tile_base, int tile_rows, int max_qgroup_len, void* ws,
                      cudaStream_t st);

// fp32 doc-band kernel for the parity path (attn_band_f32.cu); head rows are the caller's.
// records (fneed > 0): per-tile split-softmax records of the full rows, (m, l, acc[64]) x H x fneed
// per tile, for the generic kernel's head-row merge.
int launch_attn_band_f32(const AttnArgs& a, int dtype, const int32_t* seq_tile_base, int tile_rows,
                         int max_qgroup_len, float* records, int fneed, cudaStream_t st);

// tcgen05 / TMEM kernel for wide bands and dense doc rows (attn_tc.cu).
size_t tc_workspace_bytes(int nseq, int T, int H, int n_global);  // n_global: QDS global doc tokens
int launch_attn_tc(const AttnArgs& a, int dtype, const int32_t* seq_tile_base,
                   const int32_t* seq_head_base, int tile_rows, int max_qgroup_len, void* ws,
                   size_t ws_bytes, cudaStream_t st);

}  // namespace sc
