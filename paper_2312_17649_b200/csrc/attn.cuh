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
  int row_begin, row_end;  // token-row range to process
  int only_group;          // -1 all groups, else only rows of that group
};

bool load_links(const int32_t* links, Links* L);
int launch_attn_generic(const AttnArgs& a, int dtype, cudaStream_t st);

// Tiled band kernel (attn_band_mma.cu).  Returns SC_ERR_UNSUPPORTED when the
// pattern/shape is outside its envelope (the caller then uses the generic kernel).
size_t band_workspace_bytes(int nseq, int T, int H, int d, int tile_rows);
int launch_attn_band(const AttnArgs& a, int dtype, const int32_t* tok_seq,
                     const int32_t* seq_tile_base, int tile_rows, void* ws, size_t ws_bytes,
                     cudaStream_t st);

}  // namespace sc
