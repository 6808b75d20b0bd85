// Attention backward for GPU fine-tuning: the adjoint of
// sc_attn_fwd for every pattern / window / padding / QDS, fp32 math.
// Replaces the reference's chain group_attention_backward ->
// attend_segments_backward -> masked_segment_softmax_backward ->
// band_scores/band_apply_backward (R/attention.py:260-269, :348-378,
// :476-507; R/band.py:239-274).
//
// Per source row i with key slots K(i) (the forward's segments; zero-logit
// padding slots join the normaliser only):
//   P_ij = exp(s_ij - lse_i),  dP_ij = dO_i . V_j,  D_i = dO_i . O_i,
//   dS_ij = P_ij (dP_ij - D_i) / scale,
//   dQ_i = sum_j dS_ij K_j,  dK_j = sum_i dS_ij Q_i,  dV_j = sum_i P_ij dO_i.
// Two gather-form kernels, no atomics, so results are bit-reproducible:
//   1. query-major, one warp per (row, head): lse_i and D_i (kept in the
//      caller's workspace), then dQ_i;
//   2. key-major, one warp per (key row, head): enumerates the source rows
//      whose slots address the key (the transposed pattern, QDS included)
//      and reduces dK_j, dV_j in registers.
// Global QDS rows attend every key densely (their windowed result is
// discarded by the reference, R/attention.py:461-470, :488-493).
#include "attn.cuh"

namespace sc {

constexpr int kBwdWarps = 4;
constexpr int kBwdMaxD = 128;
constexpr int kBwdE = kBwdMaxD / 32;

template <typename T>
__device__ __forceinline__ float dot_sv(const float* __restrict__ xs, const T* __restrict__ r, int d) {
  float acc = 0.f;
  for (int c = 0; c < d; ++c) acc = fmaf(xs[c], to_f32(r[c]), acc);
  return acc;
}

struct BwdArgs {
  AttnArgs a;
  const void* dout;
  int64_t ld_dout;
  float* dq;
  float* dk;
  float* dv;
  int64_t ld_grad;
  float2* stats;  // [T*H]: (lse, D); lse = +inf for rows without keys
};

__device__ __forceinline__ bool is_global(const AttnArgs& a, int row) {
  return a.glob_cu != nullptr && a.flags && (a.flags[row] & 1);
}

// Key rows of source row (gs, rs) of sequence j in forward slot order, 32 per call of fn(valid, key_row).
template <typename F>
__device__ __forceinline__ void for_each_key_chunk(const AttnArgs& a, const SeqGroups& g, int j, int gs, int rs,
                                                   bool src_global, int lane, F&& fn) {
  const bool qds = a.glob_cu != nullptr;
  int seg_t[4], seg_w[4], nseg = 0;
  if (src_global) {
    for (int t = 0; t < 3; ++t) { seg_t[nseg] = t; seg_w[nseg] = SC_LINK_FULL; ++nseg; }
  } else {
    for (int t = 0; t < 3; ++t) {
      const int w = a.links.w[gs][t];
      if (w != SC_LINK_NONE) { seg_t[nseg] = t; seg_w[nseg] = w; ++nseg; }
    }
    if (qds && gs == 2) { seg_t[nseg] = 3; seg_w[nseg] = SC_LINK_FULL; ++nseg; }
  }
  for (int sgi = 0; sgi < nseg; ++sgi) {
    const int tg = seg_t[sgi], w = seg_w[sgi];
    if (tg == 3) {
      const int gb = a.glob_cu[j], ge = a.glob_cu[j + 1];
      for (int base = gb; base < ge; base += 32) {
        const int idx = base + lane;
        const bool valid = idx < ge;
        fn(valid, valid ? g.start + g.off[2] + a.glob_pos[idx] : g.start);
      }
      continue;
    }
    const int len = g.len[tg];
    int lo = 0, hi = len;
    if (w >= 0) { lo = max(0, rs - w); hi = min(len, rs + w + 1); }
    const bool excl = qds && gs == 2 && tg == 2 && w >= 0;
    for (int base = lo; base < hi; base += 32) {
      const int t = base + lane;
      bool valid = t < hi;
      const int key_row = g.start + g.off[tg] + (valid ? t : lo);
      if (valid && excl && is_global(a, key_row)) valid = false;
      fn(valid, key_row);
    }
  }
}

// Kernel 1: lse_i, D_i and dQ_i, one warp per (row, head).
template <typename T>
__global__ void __launch_bounds__(kBwdWarps * 32) attn_bwd_dq_kernel(BwdArgs b) {
  __shared__ float qs_all[kBwdWarps][kBwdMaxD];
  __shared__ float do_all[kBwdWarps][kBwdMaxD];
  const AttnArgs& a = b.a;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t item = (int64_t)blockIdx.x * kBwdWarps + warp;
  const int h = (int)(item % a.H);
  const int row = (int)(item / a.H);
  if (row >= a.T) return;
  const int j = find_seq(a.cu, a.nseq, row);
  const T* Q = static_cast<const T*>(a.q);
  const T* K = static_cast<const T*>(a.k);
  const T* V = static_cast<const T*>(a.v);
  const T* O = static_cast<const T*>(a.out);
  const T* dO = static_cast<const T*>(b.dout);
  const int d = a.d, hoff = h * d;
  const SeqGroups g = seq_groups(a.cu, a.qlen, j);
  const int i = row - g.start;
  const int gs = i == 0 ? 0 : (i < 1 + g.len[1] ? 1 : 2);
  const int rs = i - g.off[gs];
  const bool src_global = gs == 2 && is_global(a, row);

  float* qs = qs_all[warp];
  float* dos = do_all[warp];
  float dpart = 0.f;
  for (int c = lane; c < d; c += 32) {
    qs[c] = to_f32(Q[(int64_t)row * a.ld + hoff + c]);
    const float go = to_f32(dO[(int64_t)row * b.ld_dout + hoff + c]);
    dos[c] = go;
    dpart = fmaf(go, to_f32(O[(int64_t)row * a.ld_out + hoff + c]), dpart);
  }
  __syncwarp();
  const float D = warp_sum(dpart);

  // row max and normaliser; zero-logit padding slots enter with logit 0
  float m = -INFINITY, lsum = 0.f;
  if (a.padding == SC_PAD_ZERO_LOGIT && !src_global) {
    int n_inv = 0;
    for (int t = 0; t < 3; ++t) {
      const int w = a.links.w[gs][t];
      if (w < 0) continue;
      const int lo = max(0, rs - w), hi = min(g.len[t], rs + w + 1);
      n_inv += (2 * w + 1) - max(0, hi - lo);
    }
    if (n_inv > 0) { m = 0.f; lsum = lane == 0 ? (float)n_inv : 0.f; }
  }
  for_each_key_chunk(a, g, j, gs, rs, src_global, lane, [&](bool valid, int key_row) {
    const float s = valid ? dot_sv<T>(qs, K + (int64_t)key_row * a.ld + hoff, d) / a.scale : -INFINITY;
    const float cmax = warp_max(s);
    if (cmax == -INFINITY) return;
    const float mnew = fmaxf(m, cmax);
    lsum = lsum * (m == -INFINITY ? 0.f : expf(m - mnew)) + (valid ? expf(s - mnew) : 0.f);
    m = mnew;
  });
  const float l = warp_sum(lsum);
  const float lse = l > 0.f ? m + logf(l) : INFINITY;
  if (lane == 0) b.stats[item] = make_float2(lse, D);

  float dq[kBwdE];
#pragma unroll
  for (int e = 0; e < kBwdE; ++e) dq[e] = 0.f;
  if (l > 0.f) {
    for_each_key_chunk(a, g, j, gs, rs, src_global, lane, [&](bool valid, int key_row) {
      float ds = 0.f;
      if (valid) {
        const float s = dot_sv<T>(qs, K + (int64_t)key_row * a.ld + hoff, d) / a.scale;
        const float p = expf(s - lse);
        ds = p * (dot_sv<T>(dos, V + (int64_t)key_row * a.ld + hoff, d) - D) / a.scale;
      }
      unsigned live = __ballot_sync(0xffffffffu, valid);
      while (live) {
        const int kk = __ffs(live) - 1;
        live &= live - 1;
        const float dsk = __shfl_sync(0xffffffffu, ds, kk);
        const T* kr = K + (int64_t)__shfl_sync(0xffffffffu, key_row, kk) * a.ld + hoff;
#pragma unroll
        for (int e = 0; e < kBwdE; ++e) {
          const int c = lane + 32 * e;
          if (c < d) dq[e] = fmaf(dsk, to_f32(kr[c]), dq[e]);
        }
      }
    });
  }
  float* dqr = b.dq + (int64_t)row * b.ld_grad + hoff;
#pragma unroll
  for (int e = 0; e < kBwdE; ++e) {
    const int c = lane + 32 * e;
    if (c < d) dqr[c] = dq[e];
  }
}

// Kernel 2: dK_j, dV_j, one warp per (key row, head), over the transposed pattern.
template <typename T>
__global__ void __launch_bounds__(kBwdWarps * 32) attn_bwd_dkv_kernel(BwdArgs b) {
  __shared__ float ks_all[kBwdWarps][kBwdMaxD];
  __shared__ float vs_all[kBwdWarps][kBwdMaxD];
  const AttnArgs& a = b.a;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t item = (int64_t)blockIdx.x * kBwdWarps + warp;
  const int h = (int)(item % a.H);
  const int krow = (int)(item / a.H);
  if (krow >= a.T) return;
  const int j = find_seq(a.cu, a.nseq, krow);
  const T* Q = static_cast<const T*>(a.q);
  const T* K = static_cast<const T*>(a.k);
  const T* V = static_cast<const T*>(a.v);
  const T* dO = static_cast<const T*>(b.dout);
  const int d = a.d, hoff = h * d;
  const SeqGroups g = seq_groups(a.cu, a.qlen, j);
  const int i = krow - g.start;
  const int tg = i == 0 ? 0 : (i < 1 + g.len[1] ? 1 : 2);
  const int r = i - g.off[tg];
  const bool qds = a.glob_cu != nullptr;
  const bool key_global = tg == 2 && is_global(a, krow);

  float* ks = ks_all[warp];
  float* vs = vs_all[warp];
  for (int c = lane; c < d; c += 32) {
    ks[c] = to_f32(K[(int64_t)krow * a.ld + hoff + c]);
    vs[c] = to_f32(V[(int64_t)krow * a.ld + hoff + c]);
  }
  __syncwarp();

  float dk[kBwdE], dv[kBwdE];
#pragma unroll
  for (int e = 0; e < kBwdE; ++e) { dk[e] = 0.f; dv[e] = 0.f; }

  // One slot of source row `src` addressing this key (valid lanes only contribute).
  auto chunk = [&](bool valid, int src) {
    float p = 0.f, ds = 0.f;
    if (valid) {
      const float2 st = b.stats[(int64_t)src * a.H + h];
      const float s = dot_sv<T>(ks, Q + (int64_t)src * a.ld + hoff, d) / a.scale;
      p = expf(s - st.x);
      ds = p * (dot_sv<T>(vs, dO + (int64_t)src * b.ld_dout + hoff, d) - st.y) / a.scale;
    }
    unsigned live = __ballot_sync(0xffffffffu, valid && p != 0.f);
    while (live) {
      const int kk = __ffs(live) - 1;
      live &= live - 1;
      const float pk = __shfl_sync(0xffffffffu, p, kk), dsk = __shfl_sync(0xffffffffu, ds, kk);
      const int sr = __shfl_sync(0xffffffffu, src, kk);
      const T* qr = Q + (int64_t)sr * a.ld + hoff;
      const T* gr = dO + (int64_t)sr * b.ld_dout + hoff;
#pragma unroll
      for (int e = 0; e < kBwdE; ++e) {
        const int c = lane + 32 * e;
        if (c < d) {
          dk[e] = fmaf(dsk, to_f32(qr[c]), dk[e]);
          dv[e] = fmaf(pk, to_f32(gr[c]), dv[e]);
        }
      }
    }
  };

  // Source groups by link (src gs -> this key's group tg).  QDS doc sources:
  // non-global rows follow the link (minus windowed doc-doc slots on global
  // keys) plus the dense globals segment; global rows attend every key.
  for (int gs = 0; gs < 3; ++gs) {
    const int w = a.links.w[gs][tg];
    const bool qds_doc = qds && gs == 2;
    if (w != SC_LINK_NONE && !(qds_doc && tg == 2 && w >= 0 && key_global)) {
      int lo = 0, hi = g.len[gs];
      if (w >= 0) { lo = max(0, r - w); hi = min(g.len[gs], r + w + 1); }
      for (int base = lo; base < hi; base += 32) {
        const int t = base + lane;
        bool valid = t < hi;
        const int src = g.start + g.off[gs] + (valid ? t : lo);
        if (valid && qds_doc && is_global(a, src)) valid = false;
        chunk(valid, src);
      }
    }
  }
  if (qds) {
    const int dlo = g.start + g.off[2], dlen = g.len[2];
    if (key_global) {  // dense globals segment of every non-global doc row
      for (int base = 0; base < dlen; base += 32) {
        const int t = base + lane;
        const int src = dlo + min(t, dlen - 1);
        chunk(t < dlen && !is_global(a, src), src);
      }
    }
    // global doc rows attend every key of every group
    const int gb = a.glob_cu[j], ge = a.glob_cu[j + 1];
    for (int base = gb; base < ge; base += 32) {
      const int idx = base + lane;
      const bool valid = idx < ge;
      chunk(valid, valid ? dlo + a.glob_pos[idx] : dlo);
    }
  }

  float* dkr = b.dk + (int64_t)krow * b.ld_grad + hoff;
  float* dvr = b.dv + (int64_t)krow * b.ld_grad + hoff;
#pragma unroll
  for (int e = 0; e < kBwdE; ++e) {
    const int c = lane + 32 * e;
    if (c < d) { dkr[c] = dk[e]; dvr[c] = dv[e]; }
  }
}

}  // namespace sc

using namespace sc;

extern "C" size_t sc_attn_bwd_workspace_bytes(int32_t total_tokens, int32_t heads) {
  return (size_t)(total_tokens > 0 ? total_tokens : 0) * (size_t)(heads > 0 ? heads : 0) * sizeof(float2);
}

extern "C" int sc_attn_bwd(const void* q, const void* k, const void* v, int64_t row_stride, const void* out,
                           int64_t out_row_stride, const void* dout, int64_t dout_row_stride, float* dq, float* dk,
                           float* dv, int64_t grad_row_stride, const int32_t* cu_seqlens, const int32_t* qgroup_len,
                           int32_t nseq, int32_t total_tokens, int32_t heads, int32_t head_dim, const int32_t* links,
                           int32_t padding, float scale, int32_t dtype, const uint8_t* tok_flags,
                           const int32_t* glob_cu, const int32_t* glob_pos, void* workspace, size_t workspace_bytes,
                           void* stream) {
  BwdArgs b = {};
  AttnArgs& a = b.a;
  SC_CHECK_ARG(load_links(links, &a.links), "sc_attn_bwd: bad links");
  SC_CHECK_ARG(q && k && v && out && dout && dq && dk && dv && cu_seqlens && qgroup_len, "sc_attn_bwd: null pointer");
  SC_CHECK_ARG(nseq >= 1 && total_tokens >= 3 * nseq, "sc_attn_bwd: bad nseq/total_tokens");
  SC_CHECK_ARG(heads >= 1 && head_dim >= 1 && head_dim <= kBwdMaxD, "sc_attn_bwd: head_dim must be in [1,128]");
  SC_CHECK_ARG(grad_row_stride >= (int64_t)heads * head_dim, "sc_attn_bwd: gradient row stride too small");
  SC_CHECK_ARG(padding == SC_PAD_EXCLUDE || padding == SC_PAD_ZERO_LOGIT, "unknown padding mode %d", padding);
  SC_CHECK_ARG(scale > 0.f, "scale must be positive");
  SC_CHECK_ARG(dtype == SC_DTYPE_F32 || dtype == SC_DTYPE_BF16, "sc_attn_bwd: bad dtype %d", dtype);
  SC_CHECK_ARG((glob_cu == nullptr) == (glob_pos == nullptr) && (glob_cu == nullptr || tok_flags != nullptr),
               "sc_attn_bwd: QDS globals need tok_flags, glob_cu and glob_pos");
  SC_CHECK_ARG(workspace && workspace_bytes >= sc_attn_bwd_workspace_bytes(total_tokens, heads),
               "sc_attn_bwd: workspace must hold sc_attn_bwd_workspace_bytes(T, H) bytes");
  a.q = q; a.k = k; a.v = v; a.ld = row_stride; a.out = const_cast<void*>(out); a.ld_out = out_row_stride;
  a.cu = cu_seqlens; a.qlen = qgroup_len; a.nseq = nseq; a.T = total_tokens; a.H = heads; a.d = head_dim;
  a.padding = padding; a.scale = scale; a.flags = tok_flags; a.glob_cu = glob_cu; a.glob_pos = glob_pos;
  b.dout = dout; b.ld_dout = dout_row_stride; b.dq = dq; b.dk = dk; b.dv = dv; b.ld_grad = grad_row_stride;
  b.stats = static_cast<float2*>(workspace);
  const int64_t items = (int64_t)total_tokens * heads;
  const unsigned blocks = (unsigned)((items + kBwdWarps - 1) / kBwdWarps);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SC_DTYPE_F32) attn_bwd_dq_kernel<float><<<blocks, kBwdWarps * 32, 0, st>>>(b);
  else attn_bwd_dq_kernel<__nv_bfloat16><<<blocks, kBwdWarps * 32, 0, st>>>(b);
  SC_CHECK_LAUNCH("attn_bwd_dq_kernel");
  if (dtype == SC_DTYPE_F32) attn_bwd_dkv_kernel<float><<<blocks, kBwdWarps * 32, 0, st>>>(b);
  else attn_bwd_dkv_kernel<__nv_bfloat16><<<blocks, kBwdWarps * 32, 0, st>>>(b);
  SC_CHECK_LAUNCH("attn_bwd_dkv_kernel");
  return SC_OK;
}
