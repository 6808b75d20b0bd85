// Tiled tensor-core attention backward for the doc band (SURVEY §8(f)-4 fast path).
//
// The generic adjoint (attn_bwd.cu) spends ~30 instructions per (row, key)
// pair; for a +-w band that is the whole cost.  Here the doc rows and doc keys
// are processed in 64-row tiles with mma.sync m16n8k16 (bf16 in, fp32
// accumulate), FlashAttention-2 style, split into two gather-form kernels so
// the result stays deterministic:
//   A (query-major, one CTA per 64 doc rows x head): recompute S over the
//     row's band keys and its head keys (cls / query group, <= 32 slots),
//     the row statistics lse_i and D_i = dO_i . O_i (stored for kernel B),
//     P, dP = dO V^T, dS = P (dP - D) / scale and dQ = dS K;
//   B (key-major, one CTA per 64 doc keys x head): S^T over the keys' band
//     sources and head sources (cls / query rows attending the doc), P^T
//     from the sources' lse, dS^T, dV = P^T dO and dK = dS^T Q.
// The cls / query rows and keys (long dense ranges) go through the generic
// kernels in head mode.  Semantics as attn_bwd.cu; the reference chain is
// R/attention.py:260-269, :348-378, :476-507 and R/band.py:239-274.
#include "attn.cuh"
#include "mma_tile.cuh"

namespace sc {
namespace bwdband {

using namespace mmat;
constexpr int TILE = 64;           // rows (kernel A) / keys (kernel B) per CTA
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

using Args = BandBwdArgs;

// Is doc position `pos` (group-relative) within a link of window w of position `r`?
__device__ __forceinline__ bool linked(int w, int r, int pos) {
  return w == SC_LINK_FULL || (w >= 0 && abs(r - pos) <= w);
}

// Kernel A: doc rows [r0, r0+64) of one sequence, one head.  NB band keys per warp, NH head-key slots.
template <int NB, int NH>
__global__ void __launch_bounds__(128) band_dq_kernel(Args p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int KR = 48 + NB;  // band key rows staged per CTA
  const int tile = blockIdx.x, h = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = find_seq(p.tile_base, p.nseq, tile);
  const SeqGroups g = seq_groups(p.cu, p.qlen, j);
  const int dlen = g.len[2], dstart = g.start + g.off[2];
  const int r0 = (tile - p.tile_base[j]) * TILE;
  const int w = p.w, hoff = h * 64;
  const int nhead = 1 + g.len[1];

  const uint32_t sQ = smem_u32(smem), sdO = sQ + TILE * ROWB, sK = sdO + TILE * ROWB, sV = sK + KR * ROWB,
                 sKH = sV + KR * ROWB, sVH = sKH + NH * ROWB, sPT = sVH + NH * ROWB, sST = sPT + NH * ROWB;
  float* sD = reinterpret_cast<float*>(smem + (2 * TILE + 2 * KR + 4 * NH) * ROWB);

  // two cp.async groups: what S needs (Q, K band, head keys), then what dP needs (dO, V band,
  // head values) -- the second lands while the first is being used
  stage_rows(sQ, TILE, p.q, [&](int r) {
    return r0 + r < dlen ? p.q + (int64_t)(dstart + r0 + r) * p.ld + hoff : nullptr; });
  stage_rows(sK, KR, p.q, [&](int r) {
    const int pos = r0 - w + r;
    return pos >= 0 && pos < dlen ? p.k + (int64_t)(dstart + pos) * p.ld + hoff : nullptr; });
  stage_rows(sKH, NH, p.q, [&](int r) { return r < nhead ? p.k + (int64_t)(g.start + r) * p.ld + hoff : nullptr; });
  cp_async_commit();
  stage_rows(sdO, TILE, p.q, [&](int r) {
    return r0 + r < dlen ? p.dout + (int64_t)(dstart + r0 + r) * p.ld_dout + hoff : nullptr; });
  stage_rows(sV, KR, p.q, [&](int r) {
    const int pos = r0 - w + r;
    return pos >= 0 && pos < dlen ? p.v + (int64_t)(dstart + pos) * p.ld + hoff : nullptr; });
  stage_rows(sVH, NH, p.q, [&](int r) { return r < nhead ? p.v + (int64_t)(g.start + r) * p.ld + hoff : nullptr; });
  cp_async_commit();
  cp_async_wait_group<1>();
  __syncthreads();

  const int gq = lane >> 2, tq = lane & 3;
  const int ra = 16 * warp + gq;         // tile-relative rows of this thread: ra, ra + 8
  const int rsA = r0 + ra, rsB = rsA + 8;  // doc-relative
  const float c2 = p.inv_scale * LOG2E;
  constexpr int NT = NB / 8, NHT = NH / 8;

  uint32_t qa[4][4];
  load_a(sQ, 16 * warp, lane, qa);
  float s[NT][4], sh[NHT][4];
#pragma unroll
  for (int i = 0; i < NT; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
  for (int i = 0; i < NHT; ++i) sh[i][0] = sh[i][1] = sh[i][2] = sh[i][3] = 0.f;
#pragma unroll
  for (int kp = 0; kp < NB / 16; ++kp) mm_nt16(sK, 16 * warp + 16 * kp, lane, qa, s[2 * kp], s[2 * kp + 1]);
#pragma unroll
  for (int kp = 0; kp < NH / 16; ++kp) mm_nt16(sKH, 16 * kp, lane, qa, sh[2 * kp], sh[2 * kp + 1]);

  // masks: band key kb of this warp sits at doc position r0 + 16*warp - w + kb
  const int kpos0 = r0 + 16 * warp - w;
  const int L20 = p.links.w[2][0], L21 = p.links.w[2][1];
  auto band_ok = [&](int rs, int kb) {
    const int kp = kpos0 + kb;
    return rs < dlen && kp >= 0 && kp < dlen && abs(kp - rs) <= w;
  };
  auto head_ok = [&](int rs, int sl) {
    if (rs >= dlen || sl >= nhead) return false;
    return sl == 0 ? linked(L20, rs, 0) : linked(L21, rs, sl - 1);
  };
  float mA = -INFINITY, mB = -INFINITY;
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int rs = e < 2 ? rsA : rsB, kb = 8 * i + 2 * tq + (e & 1);
      s[i][e] = band_ok(rs, kb) ? s[i][e] * c2 : -INFINITY;
      if (e < 2) mA = fmaxf(mA, s[i][e]); else mB = fmaxf(mB, s[i][e]);
    }
#pragma unroll
  for (int i = 0; i < NHT; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int rs = e < 2 ? rsA : rsB, sl = 8 * i + 2 * tq + (e & 1);
      sh[i][e] = head_ok(rs, sl) ? sh[i][e] * c2 : -INFINITY;
      if (e < 2) mA = fmaxf(mA, sh[i][e]); else mB = fmaxf(mB, sh[i][e]);
    }
  mA = fmaxf(mA, __shfl_xor_sync(0xffffffffu, mA, 1));
  mA = fmaxf(mA, __shfl_xor_sync(0xffffffffu, mA, 2));
  mB = fmaxf(mB, __shfl_xor_sync(0xffffffffu, mB, 1));
  mB = fmaxf(mB, __shfl_xor_sync(0xffffffffu, mB, 2));
  // zero-logit padding: out-of-range windowed slots join with logit 0
  auto n_invalid = [&](int rs) {
    int n = 0;
    for (int t = 0; t < 3; ++t) {
      const int wt = p.links.w[2][t];
      if (wt < 0) continue;
      const int lo = max(0, rs - wt), hi = min(g.len[t], rs + wt + 1);
      n += (2 * wt + 1) - max(0, hi - lo);
    }
    return n;
  };
  const int nA = p.padding == SC_PAD_ZERO_LOGIT && rsA < dlen ? n_invalid(rsA) : 0;
  const int nB = p.padding == SC_PAD_ZERO_LOGIT && rsB < dlen ? n_invalid(rsB) : 0;
  if (nA > 0) mA = fmaxf(mA, 0.f);
  if (nB > 0) mB = fmaxf(mB, 0.f);
  const float mAs = mA == -INFINITY ? 0.f : mA, mBs = mB == -INFINITY ? 0.f : mB;
  float lA = 0.f, lB = 0.f;
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    s[i][0] = ex2(s[i][0] - mAs); s[i][1] = ex2(s[i][1] - mAs);
    s[i][2] = ex2(s[i][2] - mBs); s[i][3] = ex2(s[i][3] - mBs);
    lA += s[i][0] + s[i][1];
    lB += s[i][2] + s[i][3];
  }
#pragma unroll
  for (int i = 0; i < NHT; ++i) {
    sh[i][0] = ex2(sh[i][0] - mAs); sh[i][1] = ex2(sh[i][1] - mAs);
    sh[i][2] = ex2(sh[i][2] - mBs); sh[i][3] = ex2(sh[i][3] - mBs);
    lA += sh[i][0] + sh[i][1];
    lB += sh[i][2] + sh[i][3];
  }
  lA += __shfl_xor_sync(0xffffffffu, lA, 1);
  lA += __shfl_xor_sync(0xffffffffu, lA, 2);
  lB += __shfl_xor_sync(0xffffffffu, lB, 1);
  lB += __shfl_xor_sync(0xffffffffu, lB, 2);
  lA += nA * ex2(-mAs);
  lB += nB * ex2(-mBs);
  const float iA = lA > 0.f ? 1.f / lA : 0.f, iB = lB > 0.f ? 1.f / lB : 0.f;
  cp_async_wait_group<0>();
  __syncthreads();
  {  // D_i = dO_i . O_i, two threads per row
    const int r = threadIdx.x >> 1, half = threadIdx.x & 1;
    float acc = 0.f;
    if (r0 + r < dlen) {
      const __nv_bfloat16* orow = p.out + (int64_t)(dstart + r0 + r) * p.ld_out + hoff + half * 32;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 ov = *reinterpret_cast<const uint4*>(orow + c * 8);
        uint4 gv;
        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(gv.x), "=r"(gv.y), "=r"(gv.z), "=r"(gv.w)
                     : "r"(swz(sdO, r, half * 4 + c)));
        const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
        const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 of = __bfloat1622float2(o2[e]), gf = __bfloat1622float2(g2[e]);
          acc = fmaf(of.x, gf.x, fmaf(of.y, gf.y, acc));
        }
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (half == 0) sD[r] = acc;
  }
  __syncthreads();
  const float DA = sD[ra], DB = sD[ra + 8];
  if (tq == 0) {
    if (rsA < dlen)
      p.stats[(int64_t)(dstart + rsA) * p.H + h] =
          make_float2(lA > 0.f ? (mAs + log2f(lA)) * LN2 : INFINITY, DA);
    if (rsB < dlen)
      p.stats[(int64_t)(dstart + rsB) * p.H + h] =
          make_float2(lB > 0.f ? (mBs + log2f(lB)) * LN2 : INFINITY, DB);
  }

  // dP = dO V^T over the same slots; dS = P (dP - D) / scale (P normalised in place)
  uint32_t da[4][4];
  load_a(sdO, 16 * warp, lane, da);
  float dp[NT][4], dph[NHT][4];
#pragma unroll
  for (int i = 0; i < NT; ++i) dp[i][0] = dp[i][1] = dp[i][2] = dp[i][3] = 0.f;
#pragma unroll
  for (int i = 0; i < NHT; ++i) dph[i][0] = dph[i][1] = dph[i][2] = dph[i][3] = 0.f;
#pragma unroll
  for (int kp = 0; kp < NB / 16; ++kp) mm_nt16(sV, 16 * warp + 16 * kp, lane, da, dp[2 * kp], dp[2 * kp + 1]);
#pragma unroll
  for (int kp = 0; kp < NH / 16; ++kp) mm_nt16(sVH, 16 * kp, lane, da, dph[2 * kp], dph[2 * kp + 1]);
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    s[i][0] *= iA * (dp[i][0] - DA) * p.inv_scale; s[i][1] *= iA * (dp[i][1] - DA) * p.inv_scale;
    s[i][2] *= iB * (dp[i][2] - DB) * p.inv_scale; s[i][3] *= iB * (dp[i][3] - DB) * p.inv_scale;
  }
  const bool part = p.head_part != nullptr;
  // head-key columns, transposed into smem ([slot][row], bf16) for the per-tile head dK / dV partials
  auto st_t = [&](uint32_t buf, int sl, int row, float x) {
    const __nv_bfloat16 hv = __float2bfloat16_rn(x);
    asm volatile("st.shared.b16 [%0], %1;" ::"r"(swz(buf, sl, row >> 3) + (row & 7) * 2),
                 "h"(*reinterpret_cast<const unsigned short*>(&hv)));
  };
#pragma unroll
  for (int i = 0; i < NHT; ++i) {
    if (part) {
      const int sl = 8 * i + 2 * tq;
      st_t(sPT, sl, ra, sh[i][0] * iA); st_t(sPT, sl + 1, ra, sh[i][1] * iA);
      st_t(sPT, sl, ra + 8, sh[i][2] * iB); st_t(sPT, sl + 1, ra + 8, sh[i][3] * iB);
    }
    sh[i][0] *= iA * (dph[i][0] - DA) * p.inv_scale; sh[i][1] *= iA * (dph[i][1] - DA) * p.inv_scale;
    sh[i][2] *= iB * (dph[i][2] - DB) * p.inv_scale; sh[i][3] *= iB * (dph[i][3] - DB) * p.inv_scale;
    if (part) {
      const int sl = 8 * i + 2 * tq;
      st_t(sST, sl, ra, sh[i][0]); st_t(sST, sl + 1, ra, sh[i][1]);
      st_t(sST, sl, ra + 8, sh[i][2]); st_t(sST, sl + 1, ra + 8, sh[i][3]);
    }
  }

  // dQ = dS K
  float o[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
#pragma unroll
  for (int kp = 0; kp < NB / 16; ++kp) mm_nn16(sK, 16 * warp + 16 * kp, lane, s[2 * kp], s[2 * kp + 1], o);
#pragma unroll
  for (int kp = 0; kp < NH / 16; ++kp) mm_nn16(sKH, 16 * kp, lane, sh[2 * kp], sh[2 * kp + 1], o);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = 8 * i + 2 * tq;
    if (rsA < dlen)
      store_grad2(p.dq, (int64_t)(dstart + rsA) * p.ld_grad + hoff + c, o[i][0], o[i][1], p.grad_bf16);
    if (rsB < dlen)
      store_grad2(p.dq, (int64_t)(dstart + rsB) * p.ld_grad + hoff + c, o[i][2], o[i][3], p.grad_bf16);
  }
  if (!part) return;

  // Per-tile head-key partials: dV_h = P_h^T dO, dK_h = dS_h^T Q over this tile's 64 rows.
  // Jobs (which, n-half, m-tile) spread over the warps; summed per sequence by head_part_reduce.
  __syncthreads();
  for (int job = warp; job < 4 * (NH / 16); job += 4) {
    const int which = job & 1, nh = (job >> 1) & 1, mt = job >> 2;
    uint32_t a[4][4];
    load_a(which ? sST : sPT, 16 * mt, lane, a);
    const uint32_t bbuf = which ? sQ : sdO;
    float acc[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x) acc[x][0] = acc[x][1] = acc[x][2] = acc[x][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
      for (int q2 = 0; q2 < 2; ++q2) {
        uint32_t b[4];
        ldsm_x4_t(swz(bbuf, 16 * ks + (lane & 7) + (((lane >> 3) & 1) << 3), (2 * nh + q2) * 2 + (lane >> 4)), b);
        mma16816(acc[2 * q2], a[ks], b[0], b[1]);
        mma16816(acc[2 * q2 + 1], a[ks], b[2], b[3]);
      }
    }
    float* dst = p.head_part + (((int64_t)tile * p.H + h) * 2 + which) * NH * 64;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int c = 8 * (4 * nh + x) + 2 * tq, sl = 16 * mt + gq;
      *reinterpret_cast<float2*>(dst + sl * 64 + c) = make_float2(acc[x][0], acc[x][1]);
      *reinterpret_cast<float2*>(dst + (sl + 8) * 64 + c) = make_float2(acc[x][2], acc[x][3]);
    }
  }
}

// dK / dV of the head keys (cls / query rows) += the sum over the sequence's doc tiles of the
// kernel-A partials, in tile order (deterministic).  One thread per (seq, head, which, slot, V dims):
// V = 4 (float4 loads) for short sequences, V = 1 when many tiles per sequence need more threads.
template <int NH, int V>
__global__ void __launch_bounds__(256) head_part_reduce_kernel(Args p) {
  constexpr int G = 64 / V;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int dim = (int)(idx % G) * V;
  int64_t r = idx / G;
  const int sl = (int)(r % NH); r /= NH;
  const int which = (int)(r & 1); r >>= 1;
  const int h = (int)(r % p.H);
  const int j = (int)(r / p.H);
  if (j >= p.nseq) return;
  if (sl >= 1 + __ldg(p.qlen + j)) return;
  const int64_t off = (int64_t)(__ldg(p.cu + j) + sl) * p.ld_grad + h * 64 + dim;
  const int64_t stride = (int64_t)p.H * 2 * NH * 64;
  const float* src = p.head_part + ((int64_t)h * 2 + which) * NH * 64 + sl * 64 + dim;
  float acc[V] = {};
  const int t0 = __ldg(p.tile_base + j), t1 = __ldg(p.tile_base + j + 1);
#pragma unroll 8
  for (int t = t0; t < t1; ++t) {
    if constexpr (V == 4) {
      const float4 v = *reinterpret_cast<const float4*>(src + t * stride);
      acc[0] += v.x; acc[1] += v.y; acc[2] += v.z; acc[3] += v.w;
    } else {
      acc[0] += src[t * stride];
    }
  }
  void* base = which ? p.dk : p.dv;
#pragma unroll
  for (int e = 0; e < V; ++e) add_grad(base, off + e, acc[e], p.grad_bf16);
}

// Kernel B: doc keys [k0, k0+64) of one sequence, one head.  Sources: the band doc rows
// [k0 - w, k0 + 64 + w) and the head rows (cls / query) attending the doc.
template <int NB, int NH>
__global__ void __launch_bounds__(128, 4) band_dkv_kernel(Args p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int KR = 48 + NB;
  const int tile = blockIdx.x, h = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = find_seq(p.tile_base, p.nseq, tile);
  const SeqGroups g = seq_groups(p.cu, p.qlen, j);
  const int dlen = g.len[2], dstart = g.start + g.off[2];
  const int k0 = (tile - p.tile_base[j]) * TILE;
  const int w = p.w, hoff = h * 64;
  const int nhead = 1 + g.len[1];

  const uint32_t sK = smem_u32(smem), sV = sK + TILE * ROWB, sQ = sV + TILE * ROWB, sdO = sQ + KR * ROWB,
                 sQH = sdO + KR * ROWB, sdOH = sQH + NH * ROWB;
  float2* sSt = reinterpret_cast<float2*>(smem + (2 * TILE + 2 * KR + 2 * NH) * ROWB);  // [KR + NH]

  stage_rows(sK, TILE, p.q, [&](int r) {
    return k0 + r < dlen ? p.k + (int64_t)(dstart + k0 + r) * p.ld + hoff : nullptr; });
  stage_rows(sQ, KR, p.q, [&](int r) {
    const int pos = k0 - w + r;
    return pos >= 0 && pos < dlen ? p.q + (int64_t)(dstart + pos) * p.ld + hoff : nullptr; });
  stage_rows(sQH, NH, p.q, [&](int r) { return r < nhead ? p.q + (int64_t)(g.start + r) * p.ld + hoff : nullptr; });
  cp_async_commit();
  stage_rows(sV, TILE, p.q, [&](int r) {
    return k0 + r < dlen ? p.v + (int64_t)(dstart + k0 + r) * p.ld + hoff : nullptr; });
  stage_rows(sdO, KR, p.q, [&](int r) {
    const int pos = k0 - w + r;
    return pos >= 0 && pos < dlen ? p.dout + (int64_t)(dstart + pos) * p.ld_dout + hoff : nullptr; });
  stage_rows(sdOH, NH, p.q, [&](int r) {
    return r < nhead ? p.dout + (int64_t)(g.start + r) * p.ld_dout + hoff : nullptr; });
  cp_async_commit();
  for (int r = threadIdx.x; r < KR + NH; r += blockDim.x) {
    float2 st = make_float2(INFINITY, 0.f);
    if (r < KR) {
      const int pos = k0 - w + r;
      if (pos >= 0 && pos < dlen) st = p.stats[(int64_t)(dstart + pos) * p.H + h];
    } else if (r - KR < nhead) {
      st = p.stats[(int64_t)(g.start + r - KR) * p.H + h];
    }
    st.x *= LOG2E;  // lse in log2 units
    sSt[r] = st;
  }
  cp_async_wait_group<1>();
  __syncthreads();

  const int gq = lane >> 2, tq = lane & 3;
  const int kA = k0 + 16 * warp + gq, kB = kA + 8;  // doc-relative keys of this thread
  const float c2 = p.inv_scale * LOG2E;
  constexpr int NT = NB / 8, NHT = NH / 8;

  uint32_t ka[4][4];
  load_a(sK, 16 * warp, lane, ka);
  float s[NT][4], sh[NHT][4];
#pragma unroll
  for (int i = 0; i < NT; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
  for (int i = 0; i < NHT; ++i) sh[i][0] = sh[i][1] = sh[i][2] = sh[i][3] = 0.f;
#pragma unroll
  for (int kp = 0; kp < NB / 16; ++kp) mm_nt16(sQ, 16 * warp + 16 * kp, lane, ka, s[2 * kp], s[2 * kp + 1]);
#pragma unroll
  for (int kp = 0; kp < NH / 16; ++kp) mm_nt16(sQH, 16 * kp, lane, ka, sh[2 * kp], sh[2 * kp + 1]);

  // source cb of this warp = doc row k0 + 16*warp - w + cb (smem row 16*warp + cb)
  const int spos0 = k0 + 16 * warp - w;
  const int L02 = p.links.w[0][2], L12 = p.links.w[1][2];
  // P^T = exp(S^T / scale - lse_src) on valid slots
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int key = e < 2 ? kA : kB, cb = 8 * i + 2 * tq + (e & 1), sp = spos0 + cb;
      const bool ok = key < dlen && sp >= 0 && sp < dlen && abs(sp - key) <= w;
      s[i][e] = ok ? ex2(s[i][e] * c2 - sSt[16 * warp + cb].x) : 0.f;
    }
#pragma unroll
  for (int i = 0; i < NHT; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int key = e < 2 ? kA : kB, sl = 8 * i + 2 * tq + (e & 1);
      const bool ok = key < dlen && sl < nhead && (sl == 0 ? linked(L02, 0, key) : linked(L12, sl - 1, key));
      sh[i][e] = ok ? ex2(sh[i][e] * c2 - sSt[KR + sl].x) : 0.f;
    }

  cp_async_wait_group<0>();
  __syncthreads();
  // dV = P^T dO
  float dv[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) dv[i][0] = dv[i][1] = dv[i][2] = dv[i][3] = 0.f;
#pragma unroll
  for (int kp = 0; kp < NB / 16; ++kp) mm_nn16(sdO, 16 * warp + 16 * kp, lane, s[2 * kp], s[2 * kp + 1], dv);
#pragma unroll
  for (int kp = 0; kp < NH / 16; ++kp) mm_nn16(sdOH, 16 * kp, lane, sh[2 * kp], sh[2 * kp + 1], dv);

  // dP^T = V dO^T; dS^T = P^T (dP^T - D_src) / scale
  uint32_t va[4][4];
  load_a(sV, 16 * warp, lane, va);
  float dp[NT][4], dph[NHT][4];
#pragma unroll
  for (int i = 0; i < NT; ++i) dp[i][0] = dp[i][1] = dp[i][2] = dp[i][3] = 0.f;
#pragma unroll
  for (int i = 0; i < NHT; ++i) dph[i][0] = dph[i][1] = dph[i][2] = dph[i][3] = 0.f;
#pragma unroll
  for (int kp = 0; kp < NB / 16; ++kp) mm_nt16(sdO, 16 * warp + 16 * kp, lane, va, dp[2 * kp], dp[2 * kp + 1]);
#pragma unroll
  for (int kp = 0; kp < NH / 16; ++kp) mm_nt16(sdOH, 16 * kp, lane, va, dph[2 * kp], dph[2 * kp + 1]);
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int cb = 8 * i + 2 * tq + (e & 1);
      s[i][e] *= (dp[i][e] - sSt[16 * warp + cb].y) * p.inv_scale;
    }
#pragma unroll
  for (int i = 0; i < NHT; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int sl = 8 * i + 2 * tq + (e & 1);
      sh[i][e] *= (dph[i][e] - sSt[KR + sl].y) * p.inv_scale;
    }

  // dK = dS^T Q
  float dk[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) dk[i][0] = dk[i][1] = dk[i][2] = dk[i][3] = 0.f;
#pragma unroll
  for (int kp = 0; kp < NB / 16; ++kp) mm_nn16(sQ, 16 * warp + 16 * kp, lane, s[2 * kp], s[2 * kp + 1], dk);
#pragma unroll
  for (int kp = 0; kp < NH / 16; ++kp) mm_nn16(sQH, 16 * kp, lane, sh[2 * kp], sh[2 * kp + 1], dk);

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = 8 * i + 2 * tq;
    if (kA < dlen) {
      const int64_t off = (int64_t)(dstart + kA) * p.ld_grad + hoff + c;
      store_grad2(p.dk, off, dk[i][0], dk[i][1], p.grad_bf16);
      store_grad2(p.dv, off, dv[i][0], dv[i][1], p.grad_bf16);
    }
    if (kB < dlen) {
      const int64_t off = (int64_t)(dstart + kB) * p.ld_grad + hoff + c;
      store_grad2(p.dk, off, dk[i][2], dk[i][3], p.grad_bf16);
      store_grad2(p.dv, off, dv[i][2], dv[i][3], p.grad_bf16);
    }
  }
}


// Head rows (cls + query group, <= NH) of one sequence x one head against every key of the
// sequence: S = Qh K^T on mma.sync with M = the head rows, keys in 64-row chunks dealt to the
// kHeadWarps warps round-robin (each warp stages its chunk with cp.async into its own buffer).  Pass 1:
// per-row max / sum, combined across warps in order -> lse; pass 2: P, dP = dOh V^T, dS and
// dQ_h = dS K, reduced across warps in order.  Writes the head rows' (lse, D) and dQ.

// Keys (sequence-relative) a head row attends: one interval per target group, from the link
// table -- a few integer ops per chunk instead of a group lookup per (row, key).
struct Span3 {
  int lo[3], n[3];  // keys t with (unsigned)(t - lo) < n
};
__device__ __forceinline__ Span3 head_row_span(const Args& p, const SeqGroups& g, int i, int nhead) {
  Span3 s;
  const int rs = i == 0 ? 0 : i - 1;
#pragma unroll
  for (int tg = 0; tg < 3; ++tg) {
    const int w = i == 0 ? p.links.w[0][tg] : p.links.w[1][tg];
    int a = 0, b = 0;
    if (w == SC_LINK_FULL) b = g.len[tg];
    else if (w >= 0) a = max(0, rs - w), b = min(g.len[tg], rs + w + 1);
    s.lo[tg] = g.off[tg] + a;
    s.n[tg] = i < nhead ? max(0, b - a) : 0;
  }
  return s;
}
__device__ __forceinline__ bool in_span(const Span3& s, int t) {
  return (unsigned)(t - s.lo[0]) < (unsigned)s.n[0] || (unsigned)(t - s.lo[1]) < (unsigned)s.n[1] ||
         (unsigned)(t - s.lo[2]) < (unsigned)s.n[2];
}

template <int NH, int kHeadWarps>
__global__ void __launch_bounds__(kHeadWarps * 32) head_dq_kernel(Args p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int MT = NH / 16;
  const int j = blockIdx.x, h = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const SeqGroups g = seq_groups(p.cu, p.qlen, j);
  const int slen = g.len[0] + g.len[1] + g.len[2];
  const int nhead = 1 + g.len[1];
  const int hoff = h * 64;
  const uint32_t sQ = smem_u32(smem), sdO = sQ + NH * ROWB;
  const uint32_t sKw = sdO + NH * ROWB + warp * 2 * TILE * ROWB, sVw = sKw + TILE * ROWB;
  float* red = reinterpret_cast<float*>(smem + (2 * NH + 2 * kHeadWarps * TILE) * ROWB);  // [warps][NH][2]
  float* sD = red + kHeadWarps * NH * 2;                                                  // [NH]
  float* sL = sD + NH;                                                                     // [NH] lse (log2)
  float* red_o = sL + NH;                                                                  // [warps][NH][64]
  float* sPS = red_o + kHeadWarps * NH * 64;  // [2][NH][64]: P and dS of key chunk 0 (the head keys)
  const bool head_keys = p.head_part != nullptr;  // also write the head keys' dK/dV from head sources

  stage_rows(sQ, NH, p.q, [&](int r) { return r < nhead ? p.q + (int64_t)(g.start + r) * p.ld + hoff : nullptr; });
  stage_rows(sdO, NH, p.q, [&](int r) {
    return r < nhead ? p.dout + (int64_t)(g.start + r) * p.ld_dout + hoff : nullptr; });
  cp_async_wait_all();
  __syncthreads();
  // D_i = dO_i . O_i: eight threads per row
  for (int r = threadIdx.x >> 3; r < NH; r += kHeadWarps * 4) {
    const int part = threadIdx.x & 7;
    float acc = 0.f;
    if (r < nhead) {
      const uint4 ov = *reinterpret_cast<const uint4*>(p.out + (int64_t)(g.start + r) * p.ld_out + hoff + part * 8);
      uint4 gv;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(gv.x), "=r"(gv.y), "=r"(gv.z), "=r"(gv.w)
                   : "r"(swz(sdO, r, part)));
      const __nv_bfloat162* o2 = reinterpret_cast<const __nv_bfloat162*>(&ov);
      const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 of = __bfloat1622float2(o2[e]), gf = __bfloat1622float2(g2[e]);
        acc = fmaf(of.x, gf.x, fmaf(of.y, gf.y, acc));
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    if (part == 0) sD[r] = acc;
  }

  const int gq = lane >> 2, tq = lane & 3;
  const float c2 = p.inv_scale * LOG2E;
  uint32_t qa[MT][4][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) load_a(sQ, 16 * mt, lane, qa[mt]);
  auto stage_chunk = [&](uint32_t buf, const __nv_bfloat16* base, int k0) {
    __syncwarp();  // the previous chunk's ldmatrix reads of this buffer precede the refill
    for (int idx = lane; idx < TILE * 8; idx += 32) {
      const int r = idx >> 3, c = idx & 7;
      const bool in = k0 + r < slen;
      cp_async16(swz(buf, r, c), in ? base + (int64_t)(g.start + k0 + r) * p.ld + hoff + c * 8 : p.q, in ? 16 : 0);
    }
    cp_async_wait_all();
    __syncwarp();
  };
  const int nchunks = (slen + TILE - 1) / TILE;

  // pass 1: per-row max and sum (rows 16 mt + gq and + 8 of each m-tile)
  float m[MT][2], l[MT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) m[mt][0] = m[mt][1] = -INFINITY, l[mt][0] = l[mt][1] = 0.f;
  const int KS = p.head_ks, ks = blockIdx.z;
  const bool split = KS > 1;
  float* part = split ? p.head_split + (((int64_t)j * p.H + h) * KS) * NH * 66 : nullptr;  // [KS][NH][66]
  if (!split || p.head_phase == 1)
  for (int ch = warp + kHeadWarps * ks; ch < nchunks; ch += kHeadWarps * KS) {
    const int k0 = ch * TILE;
    stage_chunk(sKw, p.k, k0);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      float sv[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) sv[i][0] = sv[i][1] = sv[i][2] = sv[i][3] = 0.f;
#pragma unroll
      for (int kp = 0; kp < 4; ++kp) mm_nt16(sKw, 16 * kp, lane, qa[mt], sv[2 * kp], sv[2 * kp + 1]);
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int i = 16 * mt + gq + 8 * hr;
        const Span3 sp = head_row_span(p, g, i, nhead);
        float cm = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int t = k0 + 8 * nt + 2 * tq + e;
            sv[nt][2 * hr + e] = in_span(sp, t) ? sv[nt][2 * hr + e] * c2 : -INFINITY;
            cm = fmaxf(cm, sv[nt][2 * hr + e]);
          }
        cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 1));
        cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 2));
        // (no early exit: the shuffles below need the whole warp)
        const float mn = fmaxf(m[mt][hr], cm);
        const float ms = mn == -INFINITY ? 0.f : mn;
        float cs = 0.f;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) cs += ex2(sv[nt][2 * hr] - ms) + ex2(sv[nt][2 * hr + 1] - ms);
        cs += __shfl_xor_sync(0xffffffffu, cs, 1);
        cs += __shfl_xor_sync(0xffffffffu, cs, 2);
        if (cm != -INFINITY) {
          l[mt][hr] = l[mt][hr] * (m[mt][hr] == -INFINITY ? 0.f : ex2(m[mt][hr] - mn)) + cs;
          m[mt][hr] = mn;
        }
      }
    }
  }
  if (tq == 0) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int i = 16 * mt + gq + 8 * hr;
        red[(warp * NH + i) * 2] = m[mt][hr];
        red[(warp * NH + i) * 2 + 1] = l[mt][hr];
      }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NH; i += blockDim.x) {  // combine in warp order (+ zero-logit slots)
    float mm = -INFINITY, ll = 0.f;
    if (!split || p.head_phase == 1) {
      for (int w = 0; w < kHeadWarps; ++w) mm = fmaxf(mm, red[(w * NH + i) * 2]);
      for (int w = 0; w < kHeadWarps; ++w) {
        const float mw = red[(w * NH + i) * 2];
        if (mw != -INFINITY) ll += red[(w * NH + i) * 2 + 1] * ex2(mw - mm);
      }
      if (split) {  // phase 1: this split's (m, l)
        part[((int64_t)ks * NH + i) * 66] = mm;
        part[((int64_t)ks * NH + i) * 66 + 1] = ll;
        continue;
      }
    } else {  // phase 2: combine the splits in order
      for (int u = 0; u < KS; ++u) mm = fmaxf(mm, part[((int64_t)u * NH + i) * 66]);
      for (int u = 0; u < KS; ++u) {
        const float mu = part[((int64_t)u * NH + i) * 66];
        if (mu != -INFINITY) ll += part[((int64_t)u * NH + i) * 66 + 1] * ex2(mu - mm);
      }
    }
    int n_inv = 0;
    if (p.padding == SC_PAD_ZERO_LOGIT && i < nhead) {
      const int gs = i == 0 ? 0 : 1, rs = i == 0 ? 0 : i - 1;
      for (int t = 0; t < 3; ++t) {
        const int wt = p.links.w[gs][t];
        if (wt < 0) continue;
        const int lo = max(0, rs - wt), hi = min(g.len[t], rs + wt + 1);
        n_inv += (2 * wt + 1) - max(0, hi - lo);
      }
    }
    if (n_inv > 0) {
      const float mn = fmaxf(mm, 0.f);
      ll = (mm == -INFINITY ? 0.f : ll * ex2(mm - mn)) + n_inv * ex2(-mn);
      mm = mn;
    }
    const float lse2 = ll > 0.f ? mm + log2f(ll) : INFINITY;
    sL[i] = lse2;
    if (i < nhead && ks == 0) p.stats[(int64_t)(g.start + i) * p.H + h] = make_float2(lse2 * LN2, sD[i]);
  }
  if (split && p.head_phase == 1) return;
  __syncthreads();

  // pass 2: dQ_h = sum_t dS_it K_t
  uint32_t da[MT][4][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) load_a(sdO, 16 * mt, lane, da[mt]);
  float o[MT][8][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int i = 0; i < 8; ++i) o[mt][i][0] = o[mt][i][1] = o[mt][i][2] = o[mt][i][3] = 0.f;
  for (int ch = warp + kHeadWarps * ks; ch < nchunks; ch += kHeadWarps * KS) {
    const int k0 = ch * TILE;
    stage_chunk(sKw, p.k, k0);
    stage_chunk(sVw, p.v, k0);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      float sv[8][4], dp[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int e = 0; e < 4; ++e) sv[i][e] = dp[i][e] = 0.f;
#pragma unroll
      for (int kp = 0; kp < 4; ++kp) {
        mm_nt16(sKw, 16 * kp, lane, qa[mt], sv[2 * kp], sv[2 * kp + 1]);
        mm_nt16(sVw, 16 * kp, lane, da[mt], dp[2 * kp], dp[2 * kp + 1]);
      }
#pragma unroll
      for (int hr = 0; hr < 2; ++hr) {
        const int i = 16 * mt + gq + 8 * hr;
        const float lse2 = sL[i], Di = sD[i];
        const Span3 sp = head_row_span(p, g, i, nhead);
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int t = k0 + 8 * nt + 2 * tq + e;
            const float pr = in_span(sp, t) ? ex2(sv[nt][2 * hr + e] * c2 - lse2) : 0.f;
            sv[nt][2 * hr + e] = pr * (dp[nt][2 * hr + e] - Di) * p.inv_scale;
            if (head_keys && ch == 0) {  // chunk 0 holds the cls / query keys
              const int kc = 8 * nt + 2 * tq + e;
              sPS[i * 64 + kc] = pr;
              sPS[NH * 64 + i * 64 + kc] = sv[nt][2 * hr + e];
            }
          }
      }
#pragma unroll
      for (int kp = 0; kp < 4; ++kp) mm_nn16(sKw, 16 * kp, lane, sv[2 * kp], sv[2 * kp + 1], o[mt]);
    }
    if (head_keys && ch == 0) {
      // head keys t < nhead, sources = the head rows: dK_t = sum_i dS_it Q_i, dV_t = sum_i P_it dO_i
      __syncwarp();
      for (int idx = lane; idx < nhead * 64; idx += 32) {
        const int t = idx >> 6, c = idx & 63;
        float dk = 0.f, dv = 0.f;
        for (int i = 0; i < nhead; ++i) {
          uint16_t qb, gb;
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(qb) : "r"(swz(sQ, i, c >> 3) + (c & 7) * 2));
          asm volatile("ld.shared.u16 %0, [%1];" : "=h"(gb) : "r"(swz(sdO, i, c >> 3) + (c & 7) * 2));
          const float qv = __bfloat162float(*reinterpret_cast<__nv_bfloat16*>(&qb));
          const float gv = __bfloat162float(*reinterpret_cast<__nv_bfloat16*>(&gb));
          dk = fmaf(sPS[NH * 64 + i * 64 + t], qv, dk);
          dv = fmaf(sPS[i * 64 + t], gv, dv);
        }
        const int64_t off = (int64_t)(g.start + t) * p.ld_grad + hoff + c;
        store_grad(p.dk, off, dk, p.grad_bf16);
        store_grad(p.dv, off, dv, p.grad_bf16);
      }
    }
  }
  // reduce dQ over the warps in order
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int c = 8 * nt + 2 * tq, i0 = 16 * mt + gq;
      red_o[(warp * NH + i0) * 64 + c] = o[mt][nt][0];
      red_o[(warp * NH + i0) * 64 + c + 1] = o[mt][nt][1];
      red_o[(warp * NH + i0 + 8) * 64 + c] = o[mt][nt][2];
      red_o[(warp * NH + i0 + 8) * 64 + c + 1] = o[mt][nt][3];
    }
  __syncthreads();
  for (int idx = threadIdx.x; idx < NH * 64; idx += blockDim.x) {
    const int i = idx >> 6, c = idx & 63;
    if (i >= nhead) continue;
    float acc = 0.f;
    for (int w = 0; w < kHeadWarps; ++w) acc += red_o[(w * NH + i) * 64 + c];
    if (split) part[((int64_t)ks * NH + i) * 66 + 2 + c] = acc;
    else store_grad(p.dq, (int64_t)(g.start + i) * p.ld_grad + hoff + c, acc, p.grad_bf16);
  }
}

// Head-row dQ = sum of the splits' partials, in split order.
template <int NH>
__global__ void __launch_bounds__(256) head_split_reduce_kernel(Args p) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = (int)(idx & 63);
  int64_t r = idx >> 6;
  const int i = (int)(r % NH);
  r /= NH;
  const int h = (int)(r % p.H), j = (int)(r / p.H);
  if (j >= p.nseq) return;
  const SeqGroups g = seq_groups(p.cu, p.qlen, j);
  if (i >= 1 + g.len[1]) return;
  const float* part = p.head_split + (((int64_t)j * p.H + h) * p.head_ks) * NH * 66;
  float acc = 0.f;
  for (int u = 0; u < p.head_ks; ++u) acc += part[((int64_t)u * NH + i) * 66 + 2 + c];
  store_grad(p.dq, (int64_t)(g.start + i) * p.ld_grad + h * 64 + c, acc, p.grad_bf16);
}

template <int NH, int kHeadWarps>
size_t head_smem_bytes() {
  return (size_t)(2 * NH + 2 * kHeadWarps * TILE) * ROWB +
         (size_t)(kHeadWarps * NH * 2 + 2 * NH + kHeadWarps * NH * 64 + 2 * NH * 64) * sizeof(float);
}

template <int NH, int HW>
int launch_head_w(const Args& a, cudaStream_t st) {
  const size_t sm = head_smem_bytes<NH, HW>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(head_dq_kernel<NH, HW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  if (a.head_ks <= 1 || !a.head_split) {
    Args b = a;
    b.head_ks = 1;
    head_dq_kernel<NH, HW><<<dim3(a.nseq, a.H, 1), HW * 32, sm, st>>>(b);
    SC_CHECK_LAUNCH("head_dq_kernel");
    return SC_OK;
  }
  // key ranges split over head_ks CTAs per (sequence, head): (m, l) partials, then dQ partials
  // with the combined lse, then the ordered sum
  Args b = a;
  b.head_phase = 1;
  head_dq_kernel<NH, HW><<<dim3(a.nseq, a.H, a.head_ks), HW * 32, sm, st>>>(b);
  SC_CHECK_LAUNCH("head_dq_kernel");
  b.head_phase = 2;
  head_dq_kernel<NH, HW><<<dim3(a.nseq, a.H, a.head_ks), HW * 32, sm, st>>>(b);
  SC_CHECK_LAUNCH("head_dq_kernel");
  const int64_t n = (int64_t)a.nseq * a.H * NH * 64;
  head_split_reduce_kernel<NH><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(b);
  SC_CHECK_LAUNCH("head_split_reduce_kernel");
  return SC_OK;
}

// Long sequences: 8 warps per (sequence, head) share the keys; short ones (passages, a few
// 64-key chunks each): 2 warps, so several CTAs fit an SM.
template <int NH>
int launch_head(const Args& a, cudaStream_t st) {
  if (a.head_warps == 1) return launch_head_w<NH, 1>(a, st);
  return a.head_warps == 2 ? launch_head_w<NH, 2>(a, st) : launch_head_w<NH, 8>(a, st);
}

template <int NB, int NH>
size_t smem_bytes() {
  return (size_t)(2 * TILE + 2 * (48 + NB) + 4 * NH) * ROWB + (48 + NB + NH) * sizeof(float2);
}

template <int NB, int NH>
int launch_pair(const Args& a, int ntiles, int phase, cudaStream_t st) {
  const size_t sm = smem_bytes<NB, NH>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(band_dq_kernel<NB, NH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(band_dkv_kernel<NB, NH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(band_dq_kernel<NB, NH>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(band_dkv_kernel<NB, NH>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  dim3 grid(ntiles, a.H);
  if (phase == 0) {
    band_dq_kernel<NB, NH><<<grid, 128, sm, st>>>(a);
    SC_CHECK_LAUNCH("band_dq_kernel");
  } else if (phase == 2) {
    if (ntiles <= 8 * a.nseq) {  // few tiles per sequence: 4 dims per thread
      const int64_t n = (int64_t)a.nseq * a.H * 2 * NH * 16;
      head_part_reduce_kernel<NH, 4><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a);
    } else {
      const int64_t n = (int64_t)a.nseq * a.H * 2 * NH * 64;
      head_part_reduce_kernel<NH, 1><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a);
    }
    SC_CHECK_LAUNCH("head_part_reduce_kernel");
  } else {
    band_dkv_kernel<NB, NH><<<grid, 128, sm, st>>>(a);
    SC_CHECK_LAUNCH("band_dkv_kernel");
  }
  return SC_OK;
}

}  // namespace bwdband

// Phases of the fast path: 0 = kernel A (doc-row stats + dQ [+ head-key partials]),
// 1 = kernel B (doc dK/dV), 2 = add the summed head-key partials into the head keys' dK/dV,
// 3 = head rows' stats + dQ (tensor cores).
int launch_attn_bwd_band(const BandBwdArgs& a, int ntiles, int max_head, int phase, cudaStream_t st) {
  using namespace bwdband;
  if (phase == 3) return max_head <= 16 ? launch_head<16>(a, st) : launch_head<32>(a, st);
  const bool wide = a.w > 8;
  if (max_head <= 16) return wide ? launch_pair<64, 16>(a, ntiles, phase, st) : launch_pair<32, 16>(a, ntiles, phase, st);
  return wide ? launch_pair<64, 32>(a, ntiles, phase, st) : launch_pair<32, 32>(a, ntiles, phase, st);
}

}  // namespace sc
