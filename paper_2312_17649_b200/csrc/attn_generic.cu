// Generic fused pattern attention: one warp per (token row, head), any
// pattern / window / padding, QDS global tokens, fp32 or bf16 I/O with fp32
// math.  This is the fp32 parity path and the fallback for rows the tiled
// band kernel does not cover.
//
// Semantics (per source row, R/attention.py:416-473 + :290-345 + :228-257):
//   segments = pattern targets of the row's group, in order; windowed
//   segment keys t with |t - r| <= w, 0 <= t < len(target) (R/band.py:48-52);
//   QDS: doc rows add a dense segment over the doc globals and drop band
//   slots that hit a global (R/attention.py:403-413, :446-459); global doc
//   rows attend every group densely (:461-470).
//   exclude:    softmax over valid keys (error if none, R/attention.py:250-251)
//   zero-logit: out-of-range band slots join the softmax with logit 0 and a
//               zero value row (R/attention.py:244-247).
// One online softmax over the union of segments replaces the reference's
// materialised score blocks; the output equals sum_seg P_seg V_seg / Z.
#include "attn.cuh"

namespace sc {

constexpr int kGenWarps = 4;
constexpr int kMaxD = 128;

template <typename T>
__device__ __forceinline__ float dot_row(const float* __restrict__ qs, const T* __restrict__ kr, int d) {
  float acc = 0.f;
  if constexpr (sizeof(T) == 2) {
    if ((d & 7) == 0 && (((uintptr_t)kr) & 15) == 0) {
      const uint4* kv = reinterpret_cast<const uint4*>(kr);
      for (int c = 0; c < d / 8; ++c) {
        uint4 u = __ldg(kv + c);
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float2 f = __bfloat1622float2(b[e]);
          acc = fmaf(qs[8 * c + 2 * e], f.x, acc);
          acc = fmaf(qs[8 * c + 2 * e + 1], f.y, acc);
        }
      }
      return acc;
    }
  } else {
    if ((d & 3) == 0 && (((uintptr_t)kr) & 15) == 0) {
      const float4* kv = reinterpret_cast<const float4*>(kr);
      for (int c = 0; c < d / 4; ++c) {
        float4 f = __ldg(kv + c);
        acc = fmaf(qs[4 * c], f.x, acc);
        acc = fmaf(qs[4 * c + 1], f.y, acc);
        acc = fmaf(qs[4 * c + 2], f.z, acc);
        acc = fmaf(qs[4 * c + 3], f.w, acc);
      }
      return acc;
    }
  }
  for (int c = 0; c < d; ++c) acc = fmaf(qs[c], to_f32(kr[c]), acc);
  return acc;
}

// Online-softmax state of one warp; acc holds dims lane + 32*e.
struct OnlineState {
  float m;
  float l;  // per-lane partial denominator
  float acc[kMaxD / 32];
};

// Fold one chunk of <= 32 keys (one per lane) into the state.
template <typename T>
__device__ __forceinline__ void fold_chunk(OnlineState& st, bool valid, float s, int key_row,
                                           const T* __restrict__ V, int64_t ld, int hoff, int d,
                                           int lane) {
  float cmax = warp_max(valid ? s : -INFINITY);
  if (cmax == -INFINITY) return;
  float mnew = fmaxf(st.m, cmax);
  float alpha = st.m == -INFINITY ? 0.f : expf(st.m - mnew);
  float p = valid ? expf(s - mnew) : 0.f;
  st.l = st.l * alpha + p;
#pragma unroll
  for (int e = 0; e < kMaxD / 32; ++e) st.acc[e] *= alpha;
  st.m = mnew;
  unsigned live = __ballot_sync(0xffffffffu, p != 0.f);
  while (live) {
    int kk = __ffs(live) - 1;
    live &= live - 1;
    float pk = __shfl_sync(0xffffffffu, p, kk);
    int kr = __shfl_sync(0xffffffffu, key_row, kk);
    const T* vr = V + (int64_t)kr * ld + hoff;
#pragma unroll
    for (int e = 0; e < kMaxD / 32; ++e) {
      int c = lane + 32 * e;
      if (c < d) st.acc[e] = fmaf(pk, to_f32(vr[c]), st.acc[e]);
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kGenWarps * 32)
attn_generic_kernel(AttnArgs a) {
  __shared__ float qs_all[kGenWarps][kMaxD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t item = (int64_t)blockIdx.x * kGenWarps + warp;
  const int h = (int)(item % a.H);
  int row, j;
  if (a.head_base) {  // head-row mode: item -> (sequence, cls/query row)
    const int hr = (int)(item / a.H);
    if (hr >= a.n_head_rows || hr >= __ldg(a.head_base + a.nseq)) return;
    j = find_seq(a.head_base, a.nseq, hr);
    row = __ldg(a.cu + j) + (hr - __ldg(a.head_base + j));
  } else {
    row = a.row_begin + (int)(item / a.H);
    if (row >= a.row_end) return;
    j = find_seq(a.cu, a.nseq, row);
  }

  const T* Q = static_cast<const T*>(a.q);
  const T* K = static_cast<const T*>(a.k);
  const T* V = static_cast<const T*>(a.v);
  const int d = a.d, hoff = h * d;

  const SeqGroups g = seq_groups(a.cu, a.qlen, j);
  const int i = row - g.start;
  const int gs = i == 0 ? 0 : (i < 1 + g.len[1] ? 1 : 2);
  const int rs = i - g.off[gs];
  const bool qds = a.glob_cu != nullptr;
  const bool src_global = qds && gs == 2 && a.flags && (a.flags[row] & 1);

  float* qs = qs_all[warp];
  for (int c = lane; c < d; c += 32) qs[c] = to_f32(Q[(int64_t)row * a.ld + hoff + c]);
  __syncwarp();

  // Segment list: (target group, window) in pattern order, plus the QDS globals segment (tgt 3).
  int seg_t[4], seg_w[4], nseg = 0;
  if (src_global) {
    for (int t = 0; t < 3; ++t) { seg_t[nseg] = t; seg_w[nseg] = SC_LINK_FULL; ++nseg; }
  } else {
    for (int t = 0; t < 3; ++t) {
      int w = a.links.w[gs][t];
      if (w != SC_LINK_NONE) { seg_t[nseg] = t; seg_w[nseg] = w; ++nseg; }
    }
    if (qds && gs == 2) { seg_t[nseg] = 3; seg_w[nseg] = SC_LINK_FULL; ++nseg; }
  }

  OnlineState st;
  st.m = -INFINITY;
  st.l = 0.f;
#pragma unroll
  for (int e = 0; e < kMaxD / 32; ++e) st.acc[e] = 0.f;

  if (a.padding == SC_PAD_ZERO_LOGIT) {
    int n_inv = 0;
    for (int sgi = 0; sgi < nseg; ++sgi) {
      int w = seg_w[sgi];
      if (w < 0) continue;
      int len = g.len[seg_t[sgi]];
      int lo = max(0, rs - w), hi = min(len, rs + w + 1);
      n_inv += (2 * w + 1) - max(0, hi - lo);
    }
    if (n_inv > 0) {  // virtual logit-0 slots with zero value rows
      st.m = 0.f;
      st.l = lane == 0 ? (float)n_inv : 0.f;
    }
  }

  for (int sgi = 0; sgi < nseg; ++sgi) {
    const int tg = seg_t[sgi], w = seg_w[sgi];
    if (tg == 3) {  // QDS globals: dense over the listed doc positions
      const int gb = a.glob_cu[j], ge = a.glob_cu[j + 1];
      for (int base = gb; base < ge; base += 32) {
        int idx = base + lane;
        bool valid = idx < ge;
        int key_row = valid ? g.start + g.off[2] + a.glob_pos[idx] : 0;
        float s = valid ? dot_row<T>(qs, K + (int64_t)key_row * a.ld + hoff, d) / a.scale : -INFINITY;
        fold_chunk<T>(st, valid, s, key_row, V, a.ld, hoff, d, lane);
      }
      continue;
    }
    if (tg == 2 && w == SC_LINK_FULL && a.partials && i < a.fmax) {
      // Doc keys already reduced per tile by the band kernel: merge (m, l, acc).
      // Lane-parallel: one global max over all tiles, then independent weighted sums.
      const int tb = __ldg(a.tile_base + j) * a.rec_per_tile, te = __ldg(a.tile_base + j + 1) * a.rec_per_tile;
      const int64_t rstride = (int64_t)a.H * a.fmax * (d + 2);
      const float* rec0 = a.partials + (((int64_t)tb * a.H + h) * a.fmax + i) * (d + 2);
      float mloc = -INFINITY;
      for (int t = lane; t < te - tb; t += 32) {
        const float* rec = rec0 + t * rstride;
        if (rec[1] > 0.f) mloc = fmaxf(mloc, rec[0]);
      }
      const float mtiles = warp_max(mloc);
      if (mtiles == -INFINITY) continue;
      const float mnew = fmaxf(st.m, mtiles);
      const float alpha = st.m == -INFINITY ? 0.f : expf(st.m - mnew);
      st.l *= alpha;
#pragma unroll
      for (int e = 0; e < kMaxD / 32; ++e) st.acc[e] *= alpha;
      st.m = mnew;
      for (int base = 0; base < te - tb; base += 32) {
        const int t = base + lane;
        float beta = 0.f;
        if (t < te - tb) {
          const float* rec = rec0 + t * rstride;
          const float lt = rec[1];
          if (lt > 0.f) {
            beta = expf(rec[0] - mnew);
            st.l = fmaf(beta, lt, st.l);
          }
        }
        const int cnt = min(32, te - tb - base);
        for (int kk = 0; kk < cnt; ++kk) {
          const float b = __shfl_sync(0xffffffffu, beta, kk);
          const float* rec = rec0 + (base + kk) * rstride + 2;
#pragma unroll
          for (int e = 0; e < kMaxD / 32; ++e) {
            int c = lane + 32 * e;
            if (c < d && b != 0.f) st.acc[e] = fmaf(b, rec[c], st.acc[e]);
          }
        }
      }
      continue;
    }
    const int len = g.len[tg];
    int lo = 0, hi = len;
    if (w >= 0) { lo = max(0, rs - w); hi = min(len, rs + w + 1); }
    const bool excl = qds && gs == 2 && tg == 2 && w >= 0;
    for (int base = lo; base < hi; base += 32) {
      int t = base + lane;
      bool valid = t < hi;
      int key_row = g.start + g.off[tg] + (valid ? t : lo);
      if (valid && excl && a.flags && (a.flags[key_row] & 1)) valid = false;
      float s = valid ? dot_row<T>(qs, K + (int64_t)key_row * a.ld + hoff, d) / a.scale : -INFINITY;
      fold_chunk<T>(st, valid, s, key_row, V, a.ld, hoff, d, lane);
    }
  }

  float l = warp_sum(st.l);
  T* O = static_cast<T*>(a.out) + (int64_t)row * a.ld_out + hoff;
  if (l == 0.f) {
    if (lane == 0 && a.status) atomicOr(a.status, 1);
    for (int c = lane; c < d; c += 32) O[c] = from_f32<T>(0.f);
    return;
  }
  float inv = 1.f / l;
#pragma unroll
  for (int e = 0; e < kMaxD / 32; ++e) {
    int c = lane + 32 * e;
    if (c < d) O[c] = from_f32<T>(st.acc[e] * inv);
  }
}

int launch_attn_generic(const AttnArgs& a, int dtype, cudaStream_t st) {
  int64_t rows = a.head_base ? a.n_head_rows : (a.row_end - a.row_begin);
  int64_t items = rows * a.H;
  if (items <= 0) return SC_OK;
  unsigned blocks = (unsigned)((items + kGenWarps - 1) / kGenWarps);
  if (dtype == SC_DTYPE_F32)
    attn_generic_kernel<float><<<blocks, kGenWarps * 32, 0, st>>>(a);
  else
    attn_generic_kernel<__nv_bfloat16><<<blocks, kGenWarps * 32, 0, st>>>(a);
  SC_CHECK_LAUNCH("attn_generic_kernel");
  return SC_OK;
}

}  // namespace sc
