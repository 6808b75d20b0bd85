// sc_attn_fwd: argument validation and kernel dispatch for the fused
// asymmetric windowed attention (R/attention.py:416-537).
#include "attn.cuh"

using namespace sc;

extern "C" size_t sc_attn_workspace_bytes_qds(int32_t nseq, int32_t total_tokens, int32_t heads,
                                              int32_t head_dim, int32_t tile_rows, int32_t max_qgroup_len,
                                              const int32_t* links, int32_t n_global_tokens) {
  Links L;
  if (!load_links(links, &L) || n_global_tokens < 0) return 0;
  const size_t band = band_workspace_bytes(nseq, total_tokens, heads, head_dim, tile_rows, max_qgroup_len, L);
  // the tcgen05 path uses [band records | tile prefixes | QDS compact q/k/v rows]
  return ((band + 255) & ~size_t(255)) + tc_workspace_bytes(nseq, total_tokens, heads, n_global_tokens);
}

extern "C" size_t sc_attn_workspace_bytes(int32_t nseq, int32_t total_tokens, int32_t heads,
                                          int32_t head_dim, int32_t tile_rows,
                                          int32_t max_qgroup_len, const int32_t* links) {
  return sc_attn_workspace_bytes_qds(nseq, total_tokens, heads, head_dim, tile_rows, max_qgroup_len, links, 0);
}

// AUTO kernel choice by doc window: the mma.sync band kernel while the band is
// narrow (HBM-bound regime), the tcgen05 kernel once it is a dense contraction.
// Crossover measured on B200 (s=4099, H=12, 64 sequences, us/seq-layer, round 2):
// band 5.4 / 6.9 / 11.6 / 15.8 vs tcgen05 9.8 / 10.8 / 10.8 / 10.8 at w = 24 / 40 / 48 / 64;
// the band kernel's cost steps with ceil((16+2w)/32) key chunks, so it keeps w <= 40 (three).
static constexpr int kBandMaxWindow = 40;  // measured crossover (round 2): band 6.9 us at w=40, tcgen05 10.8 vs band 11.6 at w=48

extern "C" int sc_attn_fwd(const void* q, const void* k, const void* v, int64_t row_stride,
                           void* out, int64_t out_row_stride, const int32_t* cu_seqlens,
                           const int32_t* qgroup_len, int32_t nseq, int32_t total_tokens,
                           int32_t heads, int32_t head_dim, const int32_t* links, int32_t padding,
                           float scale, int32_t dtype, const int32_t* tok_seq,
                           const int32_t* seq_tile_base, const int32_t* seq_head_base,
                           int32_t tile_rows, int32_t max_qgroup_len, const uint8_t* tok_flags,
                           const int32_t* glob_cu, const int32_t* glob_pos, int32_t algo,
                           void* workspace, size_t workspace_bytes, int32_t* status,
                           void* stream) {
  (void)tok_seq;
  AttnArgs a = {};
  SC_CHECK_ARG(load_links(links, &a.links), "sc_attn_fwd: bad links");
  SC_CHECK_ARG(q && k && v && out && cu_seqlens && qgroup_len, "sc_attn_fwd: null pointer");
  SC_CHECK_ARG(nseq >= 1 && total_tokens >= 3 * nseq, "sc_attn_fwd: bad nseq/total_tokens");
  SC_CHECK_ARG(heads >= 1 && head_dim >= 1 && head_dim <= 128, "sc_attn_fwd: head_dim must be in [1,128]");
  SC_CHECK_ARG(row_stride >= (int64_t)heads * head_dim && out_row_stride >= (int64_t)heads * head_dim,
               "sc_attn_fwd: row strides smaller than heads*head_dim");
  SC_CHECK_ARG(padding == SC_PAD_EXCLUDE || padding == SC_PAD_ZERO_LOGIT, "unknown padding mode %d", padding);
  SC_CHECK_ARG(scale > 0.f, "scale must be positive, got %g", (double)scale);
  SC_CHECK_ARG(dtype == SC_DTYPE_F32 || dtype == SC_DTYPE_BF16, "sc_attn_fwd: bad dtype %d", dtype);
  SC_CHECK_ARG((glob_cu == nullptr) == (glob_pos == nullptr), "sc_attn_fwd: glob_cu/glob_pos must be both set or both NULL");
  SC_CHECK_ARG(glob_cu == nullptr || tok_flags != nullptr, "sc_attn_fwd: QDS globals need tok_flags");
  SC_CHECK_ARG(algo == SC_ATTN_AUTO || algo == SC_ATTN_GENERIC || algo == SC_ATTN_BAND_MMA ||
                   algo == SC_ATTN_TC || algo == SC_ATTN_HEAD_ROWS,
               "sc_attn_fwd: bad algo %d", algo);
  SC_CHECK_ARG(max_qgroup_len >= 1, "sc_attn_fwd: max_qgroup_len must be >= 1");
  a.q = q; a.k = k; a.v = v; a.ld = row_stride; a.out = out; a.ld_out = out_row_stride;
  a.cu = cu_seqlens; a.qlen = qgroup_len; a.nseq = nseq; a.T = total_tokens; a.H = heads;
  a.d = head_dim; a.padding = padding; a.scale = scale; a.flags = tok_flags; a.glob_cu = glob_cu;
  a.glob_pos = glob_pos; a.status = status; a.row_begin = 0; a.row_end = total_tokens;
  cudaStream_t st = (cudaStream_t)stream;
  if (algo == SC_ATTN_HEAD_ROWS) {
    // cls + query-group rows only: the band kernel's head-rows mode streams every
    // doc key once for the split-softmax records; else the generic kernel per head row
    int rc = launch_attn_band(a, dtype, seq_tile_base, seq_head_base, tile_rows, max_qgroup_len, workspace,
                              workspace_bytes, st, /*doc_rows=*/false);
    if (rc != SC_ERR_UNSUPPORTED) return rc;
    SC_CHECK_ARG(seq_head_base, "sc_attn_fwd: head-rows mode needs seq_head_base");
    a.head_base = seq_head_base;
    a.n_head_rows = nseq * (1 + max_qgroup_len);
    a.partials = nullptr;
    return launch_attn_generic(a, dtype, st);
  }
  const int w = a.links.w[2][2];
  const bool narrow = w >= 0 && w <= kBandMaxWindow;
  if (dtype == SC_DTYPE_F32 && (algo == SC_ATTN_AUTO || algo == SC_ATTN_BAND_MMA) && seq_head_base) {
    // fp32 parity path: doc rows on the tiled fp32 band kernel, head rows on the generic kernel
    // full rows (cls, longformer query rows) merge per-tile records instead of rescanning the doc
    const int fneed = full_rows_needed(a.links, max_qgroup_len);
    const size_t rec_bytes = (size_t)((total_tokens + 63) / 64 + nseq) * heads * fneed * (head_dim + 2) * 4;
    const bool recs = fneed > 0 && workspace && workspace_bytes >= rec_bytes;
    int rc = launch_attn_band_f32(a, dtype, seq_tile_base, tile_rows, max_qgroup_len,
                                  recs ? static_cast<float*>(workspace) : nullptr, recs ? fneed : 0, st);
    if (rc == SC_OK) {
      AttnArgs hrow = a;
      hrow.head_base = seq_head_base;
      hrow.n_head_rows = nseq * (1 + max_qgroup_len);
      hrow.partials = recs ? static_cast<const float*>(workspace) : nullptr;
      hrow.tile_base = seq_tile_base;
      hrow.fmax = fneed;
      hrow.rec_per_tile = 1;
      return launch_attn_generic(hrow, dtype, st);
    }
    if (algo == SC_ATTN_BAND_MMA) return rc;
  }
  if (algo == SC_ATTN_BAND_MMA || (algo == SC_ATTN_AUTO && narrow)) {
    int rc = launch_attn_band(a, dtype, seq_tile_base, seq_head_base, tile_rows, max_qgroup_len,
                              workspace, workspace_bytes, st);
    if (rc != SC_ERR_UNSUPPORTED || algo == SC_ATTN_BAND_MMA) return rc;
  }
  if (algo == SC_ATTN_TC || algo == SC_ATTN_AUTO) {
    int rc = launch_attn_tc(a, dtype, seq_tile_base, seq_head_base, tile_rows, max_qgroup_len, workspace,
                            workspace_bytes, st);
    if (rc != SC_ERR_UNSUPPORTED || algo == SC_ATTN_TC) return rc;
  }
  return launch_attn_generic(a, dtype, st);
}
