// K1: device-side sub-sequence index and mask construction over the packed
// varlen layout.  Semantics follow SubsequencePartition (R/encoder.py:58-94),
// assemble_input's span convention (R/encoder.py:154-177), _locate
// (R/reference.py:22-27), band_validity (R/band.py:48-52), pattern_mask
// (R/reference.py:30-57) and qds_global_positions (R/encoder.py:180-184).
#include <stdarg.h>

#include "common.cuh"

namespace sc {

static thread_local char g_err[512] = "";
static unsigned long long g_launches = 0;

void count_launch() { __atomic_add_fetch(&g_launches, 1ULL, __ATOMIC_RELAXED); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// Single-CTA scan over sequences: doc-row tile prefix and QDS global counts.
__global__ void seq_prefix_kernel(const int32_t* __restrict__ cu, const int32_t* __restrict__ qlen,
                                  int nseq, int tile_rows, int qds_every,
                                  int32_t* __restrict__ tile_base, int32_t* __restrict__ head_base,
                                  int32_t* __restrict__ glob_cu) {
  __shared__ int32_t s_t[1024];
  __shared__ int32_t s_g[1024];
  __shared__ int32_t s_h[1024];
  int carry_t = 0, carry_g = 0, carry_h = 0;
  for (int base = 0; base < nseq; base += blockDim.x) {
    int j = base + threadIdx.x;
    int nt = 0, ng = 0, nh = 0;
    if (j < nseq) {
      nh = 1 + qlen[j];
      int s = cu[j + 1] - cu[j];
      int doc = s - 1 - qlen[j];
      nt = (doc + tile_rows - 1) / tile_rows;
      if (qds_every > 0) ng = (doc - 1) / qds_every;  // doc tokens exclude the final [SEP]
    }
    s_t[threadIdx.x] = nt;
    s_g[threadIdx.x] = ng;
    s_h[threadIdx.x] = nh;
    __syncthreads();
    // Hillis-Steele inclusive scan (blockDim <= 1024).
    for (int o = 1; o < blockDim.x; o <<= 1) {
      int at = threadIdx.x >= o ? s_t[threadIdx.x - o] : 0;
      int ag = threadIdx.x >= o ? s_g[threadIdx.x - o] : 0;
      int ah = threadIdx.x >= o ? s_h[threadIdx.x - o] : 0;
      __syncthreads();
      s_t[threadIdx.x] += at;
      s_g[threadIdx.x] += ag;
      s_h[threadIdx.x] += ah;
      __syncthreads();
    }
    if (j < nseq) {
      tile_base[j + 1] = carry_t + s_t[threadIdx.x];
      if (head_base) head_base[j + 1] = carry_h + s_h[threadIdx.x];
      if (glob_cu) glob_cu[j + 1] = carry_g + s_g[threadIdx.x];
    }
    carry_t += s_t[blockDim.x - 1];
    carry_g += s_g[blockDim.x - 1];
    carry_h += s_h[blockDim.x - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tile_base[0] = 0;
    if (head_base) head_base[0] = 0;
    if (glob_cu) glob_cu[0] = 0;
  }
}

__global__ void token_index_kernel(const int32_t* __restrict__ cu, const int32_t* __restrict__ qlen,
                                   int nseq, int T, int qds_every, int32_t* __restrict__ tok_seq,
                                   int32_t* __restrict__ tok_group, int32_t* __restrict__ tok_rel,
                                   int32_t* __restrict__ tok_pos, uint8_t* __restrict__ tok_flags,
                                   const int32_t* __restrict__ glob_cu, int32_t* __restrict__ glob_pos) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= T) return;
  int j = find_seq(cu, nseq, r);
  SeqGroups g = seq_groups(cu, qlen, j);
  int i = r - g.start;
  int grp = i == 0 ? 0 : (i < 1 + g.len[1] ? 1 : 2);
  int rel = i - g.off[grp];
  if (tok_seq) tok_seq[r] = j;
  if (tok_group) tok_group[r] = grp;
  if (tok_rel) tok_rel[r] = rel;
  if (tok_pos) tok_pos[r] = i;
  if (tok_flags) {
    uint8_t f = 0;
    if (qds_every > 0 && grp == 2 && rel < g.len[2] - 1 && (rel + 1) % qds_every == 0) {
      f = 1;
      if (glob_pos) glob_pos[glob_cu[j] + (rel + 1) / qds_every - 1] = rel;
    }
    tok_flags[r] = f;
  }
}

// The attendability predicate shared by the mask export and (in closed form)
// the attention kernels: pattern_mask's rule, R/reference.py:44-56.
__device__ __forceinline__ bool link_ok(const Links& L, int gs, int rs, bool src_global, int gt,
                                        int rt, bool tgt_global) {
  int w = L.w[gs][gt];
  bool ok = (w == SC_LINK_FULL) || (w >= 0 && abs(rt - rs) <= w);
  if (gs == 2) {
    if (src_global) ok = true;
    if (gt == 2 && tgt_global) ok = true;
  }
  return ok;
}

__global__ void mask_export_kernel(const int32_t* __restrict__ cu, const int32_t* __restrict__ qlen,
                                   int seq, int s, Links L, const uint8_t* __restrict__ flags,
                                   uint8_t* __restrict__ out) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)s * s) return;
  int i = (int)(idx / s), t = (int)(idx % s);
  SeqGroups g = seq_groups(cu, qlen, seq);
  int gs = i == 0 ? 0 : (i < 1 + g.len[1] ? 1 : 2);
  int gt = t == 0 ? 0 : (t < 1 + g.len[1] ? 1 : 2);
  bool sg = flags && gs == 2 && (flags[g.start + i] & 1);
  bool tg = flags && gt == 2 && (flags[g.start + t] & 1);
  out[idx] = link_ok(L, gs, i - g.off[gs], sg, gt, t - g.off[gt], tg) ? 1 : 0;
}

__global__ void band_validity_kernel(int rows, int w, int tlen, uint8_t* __restrict__ out) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int width = 2 * w + 1;
  if (idx >= (int64_t)rows * width) return;
  int i = (int)(idx / width), j = (int)(idx % width);
  int t = i + j - w;
  out[idx] = (t >= 0 && t < tlen) ? 1 : 0;
}

bool load_links(const int32_t* links, Links* L) {
  if (!links) return false;
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      int v = links[a * 3 + b];
      if (v < SC_LINK_NONE) return false;
      L->w[a][b] = v;
    }
  return true;
}

}  // namespace sc

using namespace sc;

extern "C" const char* sc_last_error(void) { return g_err; }

extern "C" int sc_version(void) { return 10000; }

extern "C" uint64_t sc_kernel_launches(void) { return __atomic_load_n(&g_launches, __ATOMIC_RELAXED); }

extern "C" int sc_index_build(const int32_t* cu_seqlens, const int32_t* qgroup_len, int32_t nseq,
                              int32_t total_tokens, int32_t tile_rows, int32_t qds_every,
                              int32_t* tok_seq, int32_t* tok_group, int32_t* tok_rel,
                              int32_t* tok_pos, int32_t* seq_tile_base, int32_t* seq_head_base,
                              uint8_t* tok_flags, int32_t* glob_cu, int32_t* glob_pos,
                              void* stream) {
  SC_CHECK_ARG(cu_seqlens && qgroup_len, "sc_index_build: null layout pointer");
  SC_CHECK_ARG(nseq >= 1 && total_tokens >= 3 * nseq, "sc_index_build: bad nseq/total_tokens");
  SC_CHECK_ARG(tile_rows >= 1, "sc_index_build: tile_rows must be >= 1");
  SC_CHECK_ARG(seq_tile_base, "sc_index_build: seq_tile_base required");
  SC_CHECK_ARG(qds_every >= 0, "sc_index_build: qds_every must be >= 0");
  SC_CHECK_ARG(qds_every == 0 || (tok_flags && glob_cu && glob_pos),
               "sc_index_build: qds_every > 0 needs tok_flags, glob_cu, glob_pos");
  cudaStream_t st = (cudaStream_t)stream;
  seq_prefix_kernel<<<1, 1024, 0, st>>>(cu_seqlens, qgroup_len, nseq, tile_rows, qds_every,
                                        seq_tile_base, seq_head_base,
                                        qds_every > 0 ? glob_cu : nullptr);
  SC_CHECK_LAUNCH("seq_prefix_kernel");
  token_index_kernel<<<(total_tokens + 255) / 256, 256, 0, st>>>(
      cu_seqlens, qgroup_len, nseq, total_tokens, qds_every, tok_seq, tok_group, tok_rel, tok_pos,
      tok_flags, glob_cu, glob_pos);
  SC_CHECK_LAUNCH("token_index_kernel");
  return SC_OK;
}

extern "C" int sc_mask_export(const int32_t* cu_seqlens, const int32_t* qgroup_len, int32_t nseq,
                              int32_t seq, int32_t seq_len, const int32_t* links,
                              const uint8_t* tok_flags, uint8_t* mask_out, void* stream) {
  Links L;
  SC_CHECK_ARG(load_links(links, &L), "sc_mask_export: bad links");
  SC_CHECK_ARG(seq >= 0 && seq < nseq && seq_len >= 3 && mask_out, "sc_mask_export: bad arguments");
  int64_t n = (int64_t)seq_len * seq_len;
  mask_export_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      cu_seqlens, qgroup_len, seq, seq_len, L, tok_flags, mask_out);
  SC_CHECK_LAUNCH("mask_export_kernel");
  return SC_OK;
}

extern "C" int sc_band_validity(int32_t rows, int32_t window, int32_t target_len, uint8_t* out,
                                void* stream) {
  SC_CHECK_ARG(window >= 0, "window must be a non-negative integer, got %d", window);
  SC_CHECK_ARG(rows >= 0 && target_len >= 0 && out, "sc_band_validity: bad arguments");
  int64_t n = (int64_t)rows * (2 * window + 1);
  if (n == 0) return SC_OK;
  band_validity_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      rows, window, target_len, out);
  SC_CHECK_LAUNCH("band_validity_kernel");
  return SC_OK;
}
