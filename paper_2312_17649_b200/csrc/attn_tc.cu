// Tensor-core (tcgen05 / TMEM) attention for doc rows when the band is wide
// enough to be a dense contraction (large w, w = inf, full pattern), bf16 I/O,
// fp32 accumulation in tensor memory.  SURVEY §7 step 5: "the 128-row Q tile x
// (128+2w) K tile runs as tcgen05 UMMA (bf16 -> fp32 TMEM accumulators), then a
// masked online softmax, then PV UMMA".
//
// One CTA = 128 doc rows of one sequence x one head.  Warps:
//   0-3  softmax / epilogue: thread = row; tcgen05.ld of S, mask, online
//        softmax (exp2 domain), P (bf16) written back over S in TMEM,
//        O rescale in TMEM when the row max grows, final O / l -> bf16.
//   4    TMA producer (lane 0): Q tile, the sequence's global rows (cls +
//        query group) and a ring of BN-key K/V blocks (128B-swizzled boxes);
//        all 32 lanes: the head rows (folded in, see below).
//   5    MMA issuer (one thread): S = Q K^T (SS, K-major) into TMEM, then
//        O += P V with P read from TMEM (TS) and V as an MN-major SMEM operand.
// Key blocks: the global block (cls + query keys, N = GR) then doc keys from
// r0 - ceil(w/BN)*BN (clamped at 0: BN-aligned with the tile, so the tile's own
// 128 keys are whole ring blocks) to min(n, r0+128+w) in blocks of BN.
// Semantics as the band kernel (R/band.py:48-52, R/attention.py:125-139, :228-257).
//
// Head rows (fold): the rows of the cls / query groups are computed by warp 4
// on CUDA cores while the ring streams past -- no second pass over K/V.  Rows
// with a FULL doc link (CLS; query rows under longformer / full / QDS) take a
// split-softmax record (m, l, acc) over each 64-key half of the CTA's own doc
// keys (the band kernel's record format, indexed by 64-row doc tile); the first
// tile of each sequence also computes the head rows over the global keys (final
// for rows without a doc link, else one more record), and
// merge_full_rows_kernel folds the records (R/attention.py:416-473 for the
// cls / query groups).
#include "mma_tile.cuh"
#include "tc_common.cuh"

namespace sc {
namespace tck {
using namespace tcx;

constexpr int BM = 128, D = 64;
constexpr int NTHREADS = 192;
constexpr int S_COL = 0;
// Kernel configuration.  NBUF S/P buffers of BN key columns in TMEM (NBUF = 2
// lets QK(b+2) overlap softmax(b+1)); GR global (cls + query) key rows; CTAS
// resident CTAs per SM (TMEM NBUF*BN + D columns each); NS K/V ring stages.
template <int NBUF_, int BN_, int GR_, int CTAS_, int NS_>
struct Cfg {
  static constexpr int NBUF = NBUF_, BN = BN_, GR = GR_, CTAS = CTAS_, NS = NS_;
  static constexpr int TMEM_COLS = NBUF * BN + D <= 128 ? 128 : (NBUF * BN + D <= 256 ? 256 : 512);
  static constexpr int O_COL = NBUF * BN;
};
constexpr int ROWB = 128;

struct Params {
  int nseq, H, w;  // w < 0: whole document
  int padding, link_cls, link_query;
  float c2;
  const int32_t* cu;
  const int32_t* qlen;
  const int32_t* tile_base;  // 128-row doc tiles per sequence (prefix)
  const int32_t* tile_seq;   // 128-row tile -> sequence
  // QDS (R/attention.py:403-413, :434-470).  Doc-rows pass (qds = 1): a dense
  // key segment over the sequence's global doc tokens (gathered into a compact
  // [q|k|v] buffer) and band slots hitting a global excluded.  Global-rows pass
  // (global_rows = 1): the global doc rows, queries from the compact buffer,
  // attend every key; tile_base then counts 128-row tiles over the globals.
  int qds, global_rows;
  const uint8_t* flags;      // per-token QDS global flag (bit 0)
  const int32_t* glob_cu;    // [nseq+1] prefix of global counts
  const int32_t* glob_pos;   // doc-relative positions of the globals
  __nv_bfloat16* out;
  int64_t ld_out;
  int dout;  // head_dim (32 or 64; operands are staged as 64 zero-padded dims)
  // head-row fold (fold = 1; 0 in the QDS global-rows pass)
  int fold, fneed, fmax, ntiles_max;
  int head_fast;  // grid (H, tiles) instead of (tiles, H)
  int fold_skip;  // measurement only (SC_TC_FOLD_SKIP=1): the head-row lanes skip their math (wrong head rows)
  int hl[2][2], hdoc[2];        // head group (cls, query) -> cls / query key links; FULL doc link
  const int32_t* tile64;        // 64-row doc-tile prefix (record index of a 64-key half)
  float* partials;              // records (m, l, pad, pad, acc[64]) x fmax x H per 64-row tile
};
constexpr int REC = D + 4;

template <class C>
struct Smem {
  // offsets (bytes) from the 1024-aligned base
  static constexpr int Q = 0;
  static constexpr int KG = Q + BM * ROWB;
  static constexpr int VG = KG + C::GR * ROWB;
  static constexpr int QF = VG + C::GR * ROWB;  // q rows of the head groups (TMA, 128B swizzle)
  static constexpr int KV = QF + C::GR * ROWB;  // NS x (K block, V block)
  static constexpr int STAGE = 2 * C::BN * ROWB;
  static constexpr int HST = KV + C::NS * STAGE;  // head-row softmax state: (GR/8) x 32 lanes x 20 fp32
  static constexpr int BAR = HST + (C::GR / 8) * 32 * 20 * 4;
  // barriers: qbar, full[NS], empty[NS], s_full[2], p_full[2], pv_done[2], o_final; tmem holder
  static constexpr int TOTAL = BAR + 16 * 8 + 16;
};

// Head rows on the legacy tensor-core path (warp 4, all lanes; mma.sync m16n8k16 over the same
// 128B-swizzled K / V blocks the ring holds): 16 head rows per fragment chunk, the online-softmax
// state of a 64-key half kept in shared memory between the half's ring blocks.
template <class C>
struct HeadRows {
  using SM = Smem<C>;
  const Params& p;
  uint32_t sm0;
  float* hst;
  int lane, h, j, n_doc, r0, G;
  __device__ HeadRows(const Params& p_, uint8_t* smem, uint32_t sm0_, int lane_, int h_, int j_, const SeqGroups& g,
                      int n_doc_, int r0_)
      : p(p_), sm0(sm0_), hst(reinterpret_cast<float*>(smem + SM::HST)), lane(lane_), h(h_), j(j_), n_doc(n_doc_),
        r0(r0_), G(1 + g.len[1]) {}

  // split-softmax record of fragment rows (gq, gq + 8) of chunk fc (band-kernel format)
  __device__ void write_recs(int64_t rec_idx, int fc, float m0, float m1, float l0, float l1, const float (&o)[8][4],
                             bool only_doc_linked) const {
    const int gq = lane >> 2, tq = lane & 3;
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    const float to_nat = p.c2 * 0.69314718055994530942f;  // raw logit -> natural units (1/scale)
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int f = fc * 16 + gq + 8 * half;
      if (f >= G || f >= (only_doc_linked ? p.fneed : C::GR)) continue;
      const int grp = f == 0 ? 0 : 1;
      const float mm = half ? m1 : m0, ll = half ? l1 : l0;
      if (p.hdoc[grp]) {
        float* rec = p.partials + ((rec_idx * p.H + h) * p.fmax + f) * REC;
        if (tq == 0) {
          rec[0] = ll > 0.f ? mm * to_nat : -INFINITY;
          rec[1] = ll;
        }
#pragma unroll
        for (int nb = 0; nb < 8; ++nb)
          *reinterpret_cast<float2*>(rec + 4 + nb * 8 + 2 * tq) = make_float2(o[nb][2 * half], o[nb][2 * half + 1]);
      } else if (!only_doc_linked) {  // final row (no doc link): O / l
        const float inv = ll > 0.f ? 1.f / ll : 0.f;
        uint32_t* dst = reinterpret_cast<uint32_t*>(p.out + (int64_t)(__ldg(p.cu + j) + f) * p.ld_out + h * p.dout + 2 * tq);
#pragma unroll
        for (int nb = 0; nb < 8; ++nb)
          if (nb * 8 < p.dout) dst[nb * 4] = pack_bf16(o[nb][2 * half] * inv, o[nb][2 * half + 1] * inv);
      }
    }
  }

  // First tile of the sequence: head rows over the cls + query keys (links per source group).
  __device__ void global_keys() const {
    const int gq = lane >> 2, tq = lane & 3;
    const int hl_bits = p.hl[0][0] | (p.hl[0][1] << 1) | (p.hl[1][0] << 2) | (p.hl[1][1] << 3);
#pragma unroll
    for (int fc = 0; fc < C::GR / 16; ++fc) {
      if (fc * 16 >= G) break;
      uint32_t qa[4][4];
      mmat::load_a(sm0 + SM::QF, fc * 16, lane, qa);
      float sc[C::GR / 8][4];
#pragma unroll
      for (int nb = 0; nb < C::GR / 8; ++nb) sc[nb][0] = sc[nb][1] = sc[nb][2] = sc[nb][3] = 0.f;
#pragma unroll
      for (int gc = 0; gc < C::GR / 16; ++gc) mmat::mm_nt16(sm0 + SM::KG, gc * 16, lane, qa, sc[2 * gc], sc[2 * gc + 1]);
#pragma unroll
      for (int nb = 0; nb < C::GR / 8; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int f = fc * 16 + gq + ((e >> 1) << 3);
          const int kg = nb * 8 + 2 * tq + (e & 1);
          const int grp = f == 0 ? 0 : 1;
          if (!(f < G && kg < G && ((hl_bits >> (grp * 2 + (kg == 0 ? 0 : 1))) & 1))) sc[nb][e] = -INFINITY;
        }
      float o[8][4];
#pragma unroll
      for (int nb = 0; nb < 8; ++nb) o[nb][0] = o[nb][1] = o[nb][2] = o[nb][3] = 0.f;
      float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
      mmat::softmax_update<C::GR / 8, true>(sc, p.c2, m0, m1, l0, l1, o);
#pragma unroll
      for (int gc = 0; gc < C::GR / 16; ++gc) mmat::mm_nn16(sm0 + SM::VG, gc * 16, lane, sc[2 * gc], sc[2 * gc + 1], o);
      write_recs(p.ntiles_max + j, fc, m0, m1, l0, l1, o, false);
    }
  }

  // One ring block of the CTA's own doc keys [r0 + off, r0 + off + BN) for the FULL-doc-link rows;
  // a record closes each 64-key half (state carried in shared memory between the half's blocks).
  // Keys are the MMA's M dimension (S^T = K Qf^T, O^T = V^T P^T; P^T to the B layout by movmatrix),
  // so the full rows cost one n8 column block per 8 rows: for the sparse pattern's single CLS row
  // 2 x BN/2 mma.sync per block instead of 2 x BN with the rows as a 16-row M fragment.
  __device__ void own_block(uint32_t kvbuf, int off) const {
    constexpr int BN = C::BN, MT = BN / 16;
    const int g8 = lane >> 2, t = lane & 3;
    const int k0 = r0 + off;
    const int nk = min(BN, n_doc - k0);
    const bool first = off % 64 == 0;
    const bool close = ((off + BN) % 64 == 0) || (k0 + BN >= n_doc);
    const float c2 = p.c2;
    const uint32_t vbuf = kvbuf + BN * ROWB;
    for (int fb = 0; fb < C::GR / 8; ++fb) {
      if (fb * 8 >= p.fneed || fb * 8 >= G) break;
      float* stt = hst + (fb * 32 + lane) * 20;
      float ot[4][4];
      float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
      if (first) {
#pragma unroll
        for (int k = 0; k < 4; ++k) ot[k][0] = ot[k][1] = ot[k][2] = ot[k][3] = 0.f;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 v = *reinterpret_cast<const float4*>(stt + 4 * k);
          ot[k][0] = v.x, ot[k][1] = v.y, ot[k][2] = v.z, ot[k][3] = v.w;
        }
        m0 = stt[16], m1 = stt[17], l0 = stt[18], l1 = stt[19];
      }
      uint32_t qb[4][2];  // B fragments of full rows fb*8 .. fb*8+7: k-steps 2i, 2i+1 per x4
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        uint32_t r[4];
        mmat::ldsm_x4(mmat::swz(sm0 + SM::QF, fb * 8 + (lane & 7), 4 * i + (lane >> 3)), r);
        qb[2 * i][0] = r[0]; qb[2 * i][1] = r[1]; qb[2 * i + 1][0] = r[2]; qb[2 * i + 1][1] = r[3];
      }
      float s[MT][4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        s[mt][0] = s[mt][1] = s[mt][2] = s[mt][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          uint32_t a[4];
          mmat::ldsm_x4(mmat::swz(kvbuf, mt * 16 + (lane & 15), ks * 2 + (lane >> 4)), a);
          mmat::mma16816(s[mt], a, qb[ks][0], qb[ks][1]);
        }
      }
      float x0 = -INFINITY, x1 = -INFINITY;  // column (full-row) max over the block's keys
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (mt * 16 + g8 + ((e >> 1) << 3) >= nk) s[mt][e] = -INFINITY;
          if (e & 1) x1 = fmaxf(x1, s[mt][e]);
          else x0 = fmaxf(x0, s[mt][e]);
        }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, o));
        x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, o));
      }
      const float n0 = fmaxf(m0, x0), n1 = fmaxf(m1, x1);
      const float b0 = n0 == -INFINITY ? 0.f : n0 * c2, b1 = n1 == -INFINITY ? 0.f : n1 * c2;
      const float a0 = mmat::ex2(fmaf(m0, c2, -b0)), a1 = mmat::ex2(fmaf(m1, c2, -b1));
      float r0s = 0.f, r1s = 0.f;
      uint32_t pb[MT][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        s[mt][0] = mmat::ex2(fmaf(s[mt][0], c2, -b0));
        s[mt][1] = mmat::ex2(fmaf(s[mt][1], c2, -b1));
        s[mt][2] = mmat::ex2(fmaf(s[mt][2], c2, -b0));
        s[mt][3] = mmat::ex2(fmaf(s[mt][3], c2, -b1));
        r0s += s[mt][0] + s[mt][2];
        r1s += s[mt][1] + s[mt][3];
        pb[mt][0] = mmat::movm_t(mmat::pack_bf16(s[mt][0], s[mt][1]));
        pb[mt][1] = mmat::movm_t(mmat::pack_bf16(s[mt][2], s[mt][3]));
      }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        r0s += __shfl_xor_sync(0xffffffffu, r0s, o);
        r1s += __shfl_xor_sync(0xffffffffu, r1s, o);
      }
      l0 = fmaf(l0, a0, r0s);
      l1 = fmaf(l1, a1, r1s);
      m0 = n0;
      m1 = n1;
#pragma unroll
      for (int dm = 0; dm < 4; ++dm) {
        ot[dm][0] *= a0; ot[dm][2] *= a0;
        ot[dm][1] *= a1; ot[dm][3] *= a1;
#pragma unroll
        for (int kk = 0; kk < MT; ++kk) {
          uint32_t a[4];
          mmat::ldsm_x4_t(mmat::swz(vbuf, kk * 16 + (lane & 7) + ((lane >> 4) << 3), dm * 2 + ((lane >> 3) & 1)), a);
          mmat::mma16816(ot[dm], a, pb[kk][0], pb[kk][1]);
        }
      }
      if (close) {
        const int64_t rec_idx = __ldg(p.tile64 + j) + r0 / 64 + (off + BN - 1) / 64;
        const float to_nat = c2 * 0.69314718055994530942f;  // raw logit -> natural units (1/scale)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const int f = fb * 8 + 2 * t + c;
          if (f >= G || f >= p.fneed || !p.hdoc[f == 0 ? 0 : 1]) continue;
          float* rec = p.partials + ((rec_idx * p.H + h) * p.fmax + f) * REC;
          const float ll = c ? l1 : l0;
          if (g8 == 0) {
            rec[0] = ll > 0.f ? (c ? m1 : m0) * to_nat : -INFINITY;
            rec[1] = ll;
          }
#pragma unroll
          for (int dm = 0; dm < 4; ++dm) {
            rec[4 + dm * 16 + g8] = ot[dm][c];
            rec[4 + dm * 16 + g8 + 8] = ot[dm][2 + c];
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          *reinterpret_cast<float4*>(stt + 4 * k) = make_float4(ot[k][0], ot[k][1], ot[k][2], ot[k][3]);
        stt[16] = m0, stt[17] = m1, stt[18] = l0, stt[19] = l1;
      }
    }
  }
};

template <class C>
__global__ void __launch_bounds__(NTHREADS, C::CTAS) tc_attn_kernel(
    const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKg,
    const __grid_constant__ CUtensorMap tmVg, const __grid_constant__ CUtensorMap tmK,
    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmKq,
    const __grid_constant__ CUtensorMap tmVq, const __grid_constant__ CUtensorMap tmQf, Params p) {
  using SM = Smem<C>;
  constexpr int NS = C::NS, O_COL = C::O_COL, TMEM_COLS = C::TMEM_COLS, NBUF = C::NBUF, BN = C::BN,
                GR = C::GR;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // grid (H, tiles): the 12 heads of a tile are dispatched together, so the CTAs in flight read
  // whole 4.6 KB q|k|v rows of neighbouring tiles (L2 sectors of a row are shared, halos meet)
  const int tile = p.head_fast ? blockIdx.y : blockIdx.x, h = p.head_fast ? blockIdx.x : blockIdx.y;
  if (tile >= __ldg(p.tile_base + p.nseq)) return;
  const int j = __ldg(p.tile_seq + tile);
  const SeqGroups g = seq_groups(p.cu, p.qlen, j);
  const int n_doc = g.len[2];
  const int r0 = (tile - __ldg(p.tile_base + j)) * BM;
  const int gq0 = (p.qds || p.global_rows) ? __ldg(p.glob_cu + j) : 0;  // first compact row of seq j
  const int n_gq = (p.qds || p.global_rows) ? __ldg(p.glob_cu + j + 1) - gq0 : 0;
  const int rows_here = min(BM, (p.global_rows ? n_gq : n_doc) - r0);
  const int doc0 = g.start + g.off[2];
  const int G = 1 + g.len[1];
  const bool has_glob = (p.link_cls || p.link_query);
  const int w = p.global_rows ? -1 : p.w;
  // BN-aligned with r0 (r0 is a multiple of BM): the own keys [r0, r0 + BM) are whole ring blocks
  const int lo = w < 0 ? 0 : max(0, r0 - (w + BN - 1) / BN * BN);
  const int hi = w < 0 ? n_doc : min(n_doc, r0 + rows_here + w);
  const int ngd = p.qds ? (n_gq + BN - 1) / BN : 0;  // key blocks over the compact QDS globals
  const int nkb = ngd + (hi - lo + BN - 1) / BN;       // K/V ring blocks: QDS globals, then band
  // block b: cls/query block first, then the ring blocks
  const int nblocks = (has_glob ? 1 : 0) + nkb;

  const uint32_t sm0 = smem_u32(smem);
  const uint32_t bar0 = sm0 + SM::BAR;
  // barriers: qbar | full[NS] | empty[NS] | s_full[2] | p_full[2] | pv_done[2] | o_final
  const uint32_t qbar = bar0, full_bar = bar0 + 8, empty_bar = bar0 + 8 * (1 + NS);
  const uint32_t s_full = bar0 + 8 * (1 + 2 * NS), p_full = s_full + 16, pv_done = s_full + 32,
                 o_final = s_full + 48;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + SM::BAR + 16 * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    mbar_init(qbar, 1);
    for (int s = 0; s < NS; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, p.fold ? 2 : 1);  // MMA commit (+ the head-row lanes)
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full + 8 * b, 1);
      mbar_init(p_full + 8 * b, 4);
      mbar_init(pv_done + 8 * b, 1);
    }
    mbar_init(o_final, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "n"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 4) {
    // ------------------------------------------------------------- TMA (one lane) + head rows
    auto issue = [&](int kb) {
      const int s = kb % NS;
      mbar_expect_tx(full_bar + 8 * s, SM::STAGE);
      const uint32_t kbuf = sm0 + SM::KV + s * SM::STAGE;
      if (kb < ngd) {
        tma_load_3d(kbuf, &tmKq, h, gq0 + kb * BN, full_bar + 8 * s);
        tma_load_3d(kbuf + BN * ROWB, &tmVq, h, gq0 + kb * BN, full_bar + 8 * s);
      } else {
        tma_load_3d(kbuf, &tmK, h, doc0 + lo + (kb - ngd) * BN, full_bar + 8 * s);
        tma_load_3d(kbuf + BN * ROWB, &tmV, h, doc0 + lo + (kb - ngd) * BN, full_bar + 8 * s);
      }
    };
    // The warp runs converged; one elect.sync lane issues each group of TMA loads (their operands
    // stay warp-uniform: no per-lane waterfall loop around UTMALDG).
    if (elect_one()) {
      mbar_expect_tx(qbar, (BM + (p.fold ? 3 : 2) * GR) * ROWB);
      tma_load_3d(sm0 + SM::Q, &tmQ, h, p.global_rows ? gq0 + r0 : doc0 + r0, qbar);
      tma_load_3d(sm0 + SM::KG, &tmKg, h, g.start, qbar);
      tma_load_3d(sm0 + SM::VG, &tmVg, h, g.start, qbar);
      if (p.fold) tma_load_3d(sm0 + SM::QF, &tmQf, h, g.start, qbar);
      for (int kb = 0; kb < min(NS, nkb); ++kb) issue(kb);
    }
    __syncwarp();
    if (!p.fold) {
      for (int kb = NS; kb < nkb; ++kb) {
        mbar_wait(empty_bar + 8 * (kb % NS), ((kb / NS) & 1) ^ 1);
        if (elect_one()) issue(kb);
        __syncwarp();
      }
    } else {
      const HeadRows<C> hr(p, smem, sm0, lane, h, j, g, n_doc, r0);
      const int own0 = ngd + (r0 - lo) / BN;          // first ring block of the own keys
      const int nown = (min(BM, n_doc - r0) + BN - 1) / BN;
      // Only the own-key blocks need the head-row lanes: the others are released (and their
      // refills issued) as soon as the MMA has consumed them.  The global-key rows of the first
      // tile come last, after the ring is done with this warp.
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % NS;
        const bool own = kb >= own0 && kb < own0 + nown;
        if (own) {
          mbar_wait(qbar, 0);  // QF (one-shot barrier: returns at once after the first time)
          mbar_wait(full_bar + 8 * s, (kb / NS) & 1);
          if (!p.fold_skip) hr.own_block(sm0 + SM::KV + s * SM::STAGE, (kb - own0) * BN);
        }
        __syncwarp();
        if (elect_one()) mbar_arrive(empty_bar + 8 * s);
        __syncwarp();
        if (kb + NS < nkb) {
          mbar_wait(empty_bar + 8 * s, (kb / NS) & 1);
          if (elect_one()) issue(kb + NS);
          __syncwarp();
        }
      }
      mbar_wait(qbar, 0);
      if (r0 == 0 && !p.fold_skip) hr.global_keys();
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------- MMA (one elected lane)
    // The whole warp runs the loop and the barrier waits; one elected lane issues each group of
    // tcgen05.mma + commit.  S is double-buffered in TMEM: QK(b+2) is issued as soon as PV(b)
    // has read P(b) out of the same buffer, so the tensor core runs ahead of softmax.
    {
      const uint32_t id_qk = idesc_bf16(BM, BN, 0), id_qg = idesc_bf16(BM, GR, 0),
                     id_pv = idesc_bf16(BM, D, 1);
      const uint32_t tO = tmem + O_COL;
      mbar_wait(qbar, 0);
      tc_fence_after();
      const uint64_t qd = sw128_desc(sm0 + SM::Q);
      auto issue_qk = [&](int b) {
        const uint32_t tS = tmem + S_COL + (b % NBUF) * BN;
        // one issue site for both block kinds (operands chosen first): with two tcgen05.mma
        // sites under divergent branches ptxas was seen to leave one copy's uniform operands
        // unset when GR == BN (VMID32: wrong S, or an illegal-instruction trap)
        uint32_t kaddr = sm0 + SM::KG, idq = id_qg;
        if (!(has_glob && b == 0)) {
          const int kb = b - (has_glob ? 1 : 0), s = kb % NS;
          mbar_wait(full_bar + 8 * s, (kb / NS) & 1);
          tc_fence_after();
          kaddr = sm0 + SM::KV + s * SM::STAGE;
          idq = id_qk;
        }
        const uint64_t kd = sw128_desc(kaddr);
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) mma_ss(tS, qd + 2 * ks, kd + 2 * ks, idq, ks > 0);
          tc_commit(s_full + 8 * (b % NBUF));
        }
        __syncwarp();
      };
      issue_qk(0);
      if (NBUF == 2 && nblocks > 1) issue_qk(1);
      for (int b = 0; b < nblocks; ++b) {
        const int buf = b % NBUF;
        mbar_wait(p_full + 8 * buf, (b / NBUF) & 1);
        tc_fence_after();
        const uint32_t tS = tmem + S_COL + buf * BN;
        const bool gblk = has_glob && b == 0;
        const int kb = b - (has_glob ? 1 : 0), s = kb % NS;
        const uint64_t vd = sw128_desc(gblk ? sm0 + SM::VG : sm0 + SM::KV + s * SM::STAGE + BN * ROWB);
        const int nks = gblk ? GR / 16 : BN / 16;
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < (GR > BN ? GR : BN) / 16; ++ks)
            if (ks < nks) mma_ts(tO, tS + 8 * ks, vd + 128 * ks, id_pv, (b > 0 || ks > 0));
          if (!gblk) tc_commit(empty_bar + 8 * s);
          tc_commit(pv_done + 8 * buf);
        }
        __syncwarp();
        if (b + NBUF < nblocks) {
          mbar_wait(pv_done + 8 * buf, (b / NBUF) & 1);  // P(b) consumed: S buffer free
          issue_qk(b + NBUF);
        }
      }
      if (elect_one()) tc_commit(o_final);
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------- softmax (thread = row)
    const int r = warp * 32 + lane;  // row within the tile (TMEM lane)
    const int rr = r0 + r;           // doc-relative row
    const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
    const float c2 = p.c2;
    // Lazy rescaling (FA4): the running max moves only when a block exceeds it
    // by more than 2^8 in the exp2 domain, so O is rarely touched.
    const float tau = 8.f / c2;
    float m = -INFINITY, l = 0.f;
    if (p.padding == SC_PAD_ZERO_LOGIT && w >= 0) {
      const int ninv = 2 * w + 1 - max(0, min(n_doc, rr + w + 1) - max(0, rr - w));
      if (ninv > 0) { m = 0.f; l = (float)ninv; }
    }
    for (int b = 0; b < nblocks; ++b) {
      const int buf = b % NBUF;
      const bool glob = has_glob && b == 0;
      const uint32_t sa = lane_addr + S_COL + buf * BN;
      mbar_wait(s_full + 8 * buf, (b / NBUF) & 1);
      tc_fence_after();
      // A band block no row of this warp reaches (the tile is a rectangle of keys, the band a
      // parallelogram): P = 0 for the warp's 32 lanes, no logits read, no exponentials.
      if (!glob && w >= 0 && b - (has_glob ? 1 : 0) >= ngd) {
        const int k0 = lo + (b - (has_glob ? 1 : 0) - ngd) * BN;
        if (k0 + BN - 1 < r0 + warp * 32 - w || k0 > r0 + warp * 32 + 31 + w) {
          uint32_t z[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) z[e] = 0u;
#pragma unroll
          for (int c = 0; c < BN / 2; c += 16) TC_ST16(sa + c, z);
          tc_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(p_full + 8 * buf);
          continue;
        }
      }
      uint32_t v[BN];
#pragma unroll
      for (int c0 = 0; c0 < BN; c0 += 32) TC_LD32(sa + c0, (&v[c0]));
      tc_wait_ld();
      if (glob) {
#pragma unroll
        for (int e = 0; e < BN; ++e)
          if (!(e < GR && e < G && (e == 0 ? p.link_cls : p.link_query))) v[e] = __float_as_uint(-INFINITY);
      } else if (b - (has_glob ? 1 : 0) < ngd) {
        // QDS global-doc block: compact rows gq0 + kb*BN + e, valid while < n_gq
        const int nval = n_gq - (b - (has_glob ? 1 : 0)) * BN;
#pragma unroll
        for (int e = 0; e < BN; ++e)
          if (e >= nval) v[e] = __float_as_uint(-INFINITY);
      } else {
        const int k0 = lo + (b - (has_glob ? 1 : 0) - ngd) * BN;
        bool interior =
            k0 + BN <= hi && (w < 0 || (k0 >= r0 + rows_here - 1 - w && k0 + BN - 1 <= r0 + w));
        if (p.qds) {
          // band slots that hit a global doc token are covered by the dense
          // global segment: hard-excluded in both padding modes (R/attention.py:326-331)
#pragma unroll
          for (int c0 = 0; c0 < BN; c0 += 32) {
            const int t = k0 + c0 + lane;
            const uint32_t gm = __ballot_sync(0xffffffffu, t < n_doc && (__ldg(p.flags + doc0 + t) & 1));
            if (gm) {
              interior = false;
#pragma unroll
              for (int e = 0; e < 32; ++e)
                if ((gm >> e) & 1u) v[c0 + e] = __float_as_uint(-INFINITY);
            }
          }
        }
        if (!interior) {
          // valid keys of this row in the block: e in [ea, eb) (band and document end)
          const int ea = w < 0 ? 0 : min(max(rr - w - k0, 0), BN);
          const int eb = max(min(min(hi, w < 0 ? hi : rr + w + 1) - k0, BN), ea);
#pragma unroll
          for (int c0 = 0; c0 < BN; c0 += 32) {
            const int a = min(max(ea - c0, 0), 32), z = min(max(eb - c0, 0), 32);
            const uint32_t keep = (z >= 32 ? 0xffffffffu : ((1u << z) - 1u)) & ~(a >= 32 ? 0xffffffffu : ((1u << a) - 1u));
#pragma unroll
            for (int e = 0; e < 32; ++e)
              if (!((keep >> e) & 1u)) v[c0 + e] = __float_as_uint(-INFINITY);
          }
        }
      }
      const float mx = row_max<BN>(v);
      const bool grow = mx > m + tau || (m == -INFINITY && mx != -INFINITY);
      float alpha = 1.f;
      if (__any_sync(0xffffffffu, grow)) {
        const float mnew = grow ? fmaxf(m, mx) : m;
        alpha = (grow && m != -INFINITY) ? ex2((m - mnew) * c2) : (grow ? 0.f : 1.f);
        m = mnew;
        if (b > 0) {  // O holds blocks < b: wait until PV(b-1) has landed, then rescale in TMEM
          mbar_wait(pv_done + 8 * ((b - 1) % NBUF), ((b - 1) / NBUF) & 1);
          tc_fence_after();
#pragma unroll
          for (int c0 = 0; c0 < D; c0 += 16) {  // 16-column chunks: S row stays in registers
            uint32_t o[16];
            TC_LD16(lane_addr + O_COL + c0, o);
            tc_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            TC_ST16(lane_addr + O_COL + c0, o);
          }
        }
      }
      const float base = m == -INFINITY ? 0.f : m * c2;
      const float rs = row_exp_pack<BN>(v, c2, base);
#pragma unroll
      for (int c = 0; c < BN / 2; c += 16) TC_ST16(sa + c, (&v[c]));
      l = fmaf(l, alpha, rs);
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full + 8 * buf);
    }
    // epilogue: O / l -> bf16 row
    mbar_wait(o_final, 0);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const int orow = p.global_rows ? (r < rows_here ? __ldg(p.glob_pos + gq0 + rr) : 0) : rr;
    __nv_bfloat16* dst = p.out + (int64_t)(doc0 + orow) * p.ld_out + h * p.dout;
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      if (c0 >= p.dout) break;  // head_dim 32: the zero-padded half of O stays in TMEM
      uint32_t o[32];
      TC_LD32(lane_addr + O_COL + c0, o);
      tc_wait_ld();
      if (r < rows_here) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + c0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          u.x = pack_bf16(__uint_as_float(o[8 * q + 0]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
          u.y = pack_bf16(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
          u.z = pack_bf16(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
          u.w = pack_bf16(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
          d4[q] = u;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS) : "memory");
  }
}

// 128-row tile prefix per sequence (single CTA scan): over the doc rows, or
// (glob_cu != nullptr) over the QDS global doc rows.
__global__ void tile128_prefix_kernel(const int32_t* __restrict__ cu, const int32_t* __restrict__ qlen, int nseq,
                                      const int32_t* __restrict__ glob_cu, int32_t* __restrict__ base,
                                      int32_t* __restrict__ tile_seq) {
  __shared__ int32_t s[1024];
  int carry = 0;
  for (int b = 0; b < nseq; b += blockDim.x) {
    const int j = b + threadIdx.x;
    int n = 0;
    if (j < nseq)
      n = glob_cu ? (glob_cu[j + 1] - glob_cu[j] + BM - 1) / BM : (cu[j + 1] - cu[j] - 1 - qlen[j] + BM - 1) / BM;
    s[threadIdx.x] = n;
    __syncthreads();
    for (int o = 1; o < blockDim.x; o <<= 1) {
      int a = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
      __syncthreads();
      s[threadIdx.x] += a;
      __syncthreads();
    }
    if (j < nseq) {
      base[j + 1] = carry + s[threadIdx.x];
      for (int t = carry + s[threadIdx.x] - n; t < carry + s[threadIdx.x]; ++t) tile_seq[t] = j;  // tile -> sequence
    }
    carry += s[blockDim.x - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) base[0] = 0;
}

// QDS: copy the q, k, v rows of every global doc token into the compact
// [n_glob][q | k | v] buffer (one warp per row, 16-byte vectors).
__global__ void qds_gather_kernel(const int32_t* __restrict__ cu, const int32_t* __restrict__ qlen, int nseq,
                                  const int32_t* __restrict__ glob_cu, const int32_t* __restrict__ glob_pos,
                                  const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                                  const __nv_bfloat16* __restrict__ v, int64_t ld, int hd, int cap,
                                  __nv_bfloat16* __restrict__ dst, int32_t* __restrict__ status) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  const int total = __ldg(glob_cu + nseq);
  if (i == 0 && lane == 0 && total > cap && status) *status = SC_ERR_INVALID;
  if (i >= min(total, cap)) return;
  const int j = find_seq(glob_cu, nseq, i);
  const int64_t row = (int64_t)__ldg(cu + j) + 1 + __ldg(qlen + j) + __ldg(glob_pos + i);
  const __nv_bfloat16* src[3] = {q + row * ld, k + row * ld, v + row * ld};
  __nv_bfloat16* d = dst + (int64_t)i * 3 * hd;
#pragma unroll
  for (int part = 0; part < 3; ++part)
    for (int c = lane * 8; c < hd; c += 256)
      *reinterpret_cast<uint4*>(d + part * hd + c) = __ldg(reinterpret_cast<const uint4*>(src[part] + c));
}

template <class C>
static int launch_kernel(dim3 grid, const CUtensorMap* maps, const Params& p, cudaStream_t st) {
  const size_t smem = Smem<C>::TOTAL + 1024;
  static bool attr = false;
  if (!attr) {
    // several CTAs per SM: ask for the full shared-memory carveout
    cudaFuncSetAttribute(tc_attn_kernel<C>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (cudaFuncSetAttribute(tc_attn_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess) {
      set_error("tcgen05 kernel: shared memory request of %zu bytes failed", smem);
      return SC_ERR_UNSUPPORTED;
    }
    attr = true;
  }
  tc_attn_kernel<C><<<grid, NTHREADS, smem, st>>>(maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6],
                                                  maps[7], p);
  SC_CHECK_LAUNCH("tc_attn_kernel");
  return SC_OK;
}

// Variants (NBUF, BN, GR, CTAS, NS), measured on B200 at s=4099, H=12, 64 sequences
// (us per sequence-layer, w = 64 / 256 / inf):
//   VLONG  2 x 64-key S buffers, 2 CTAs/SM                 17.8 / 23.3 / 75.5
//   VMID   2 x 32-key S buffers, 4 CTAs/SM, <= 15 globals   14.7 / 20.8 / 77.0
//   VMID32 the same with 32 global rows                     15.1 / 22.9 / 110
// (single-buffered S at 3-4 CTAs/SM: 19.0 / 26.8 / 94.6).  Four short
// softmax chains per SM beat two long ones until the key range is the whole
// document.
using VLONG = Cfg<2, 64, 32, 2, 4>;
using VMID = Cfg<2, 32, 16, 4, 3>;
using VMID32 = Cfg<2, 32, 32, 4, 2>;
using VG64 = Cfg<2, 64, 64, 2, 3>;  // query groups of 32..63 rows (64 global key rows)

}  // namespace tck

// [doc-tile prefix | global-tile prefix] (+ the compact QDS [q|k|v] rows).
// [doc-tile prefix | global-tile prefix | doc-tile -> sequence map | global-tile -> sequence map]
static int tc_max_tiles(int nseq, int T) { return (T + tck::BM - 1) / tck::BM + nseq; }
static size_t tc_prefix_bytes(int nseq, int T) {
  return ((size_t)(2 * (nseq + 1) + 2 * tc_max_tiles(nseq, T)) * sizeof(int32_t) + 255) & ~size_t(255);
}
size_t tc_workspace_bytes(int nseq, int T, int H, int n_global) {
  return tc_prefix_bytes(nseq, T) + (size_t)n_global * 3 * H * tck::D * sizeof(__nv_bfloat16);
}

int launch_attn_tc(const AttnArgs& a, int dtype, const int32_t* seq_tile_base,
                   const int32_t* seq_head_base, int tile_rows, int max_qgroup_len, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  using namespace tck;
  const Links& L = a.links;
  auto unsupported = [](const char* why) {
    set_error("tcgen05 kernel: %s", why);
    return SC_ERR_UNSUPPORTED;
  };
  const bool qds = a.glob_cu != nullptr;
  if (dtype != SC_DTYPE_BF16) return unsupported("needs bf16");
  if (a.d != D && a.d != 32) return unsupported("needs head_dim 32 or 64");
  if (qds && (!a.flags || !a.glob_pos)) return unsupported("QDS needs tok_flags and glob_pos");
  const int w = L.w[2][2];
  if (w == SC_LINK_NONE) return unsupported("doc rows must attend doc keys");
  if (qds && w == SC_LINK_FULL) return unsupported("QDS with a full doc->doc link");
  if (L.w[2][0] != SC_LINK_FULL && L.w[2][0] != SC_LINK_NONE) return unsupported("windowed doc->cls");
  if (L.w[2][1] != SC_LINK_FULL && L.w[2][1] != SC_LINK_NONE) return unsupported("windowed doc->query");
  if (max_qgroup_len + 1 > 64) return unsupported("query group longer than 63 rows");
  // head rows go through the band kernel's head-rows-only mode: same link envelope
  for (int x : {L.w[0][0], L.w[0][1], L.w[0][2], L.w[1][0], L.w[1][1], L.w[1][2]})
    if (x != SC_LINK_FULL && x != SC_LINK_NONE) return unsupported("windowed head-row link");
  if (tile_rows != 64 || !seq_tile_base || !seq_head_base) return unsupported("layout tiles must be 64 rows");
  if (((uintptr_t)a.q | (uintptr_t)a.k | (uintptr_t)a.v | (uintptr_t)a.out) & 15) return unsupported("alignment");
  if ((a.ld * 2) % 16 || (a.ld_out * 2) % 16) return unsupported("row strides");
  // workspace = [band-kernel records (head rows) | tile prefixes | QDS compact rows]
  const size_t band_bytes = (band_workspace_bytes(a.nseq, a.T, a.H, a.d, tile_rows, max_qgroup_len, L) + 255) & ~size_t(255);
  if (!ws || ws_bytes < band_bytes + tc_prefix_bytes(a.nseq, a.T)) return unsupported("workspace too small");
  const size_t row_bytes = (size_t)3 * a.H * a.d * sizeof(__nv_bfloat16);
  const int cap = qds ? (int)((ws_bytes - band_bytes - tc_prefix_bytes(a.nseq, a.T)) / row_bytes) : 0;

  // Variant choice (env SC_TC_VARIANT = 0/1/2 forces VLONG/VMID/VMID32, for measurement sweeps).
  static int forced = -2;
  if (forced == -2) {
    const char* e = getenv("SC_TC_VARIANT");
    forced = e ? atoi(e) : -1;
  }
  const bool long_range = w == SC_LINK_FULL || w > 256;
  const bool small_gr = max_qgroup_len + 1 <= 16;
  const bool big_gr = max_qgroup_len + 1 > 32;
  int var = forced >= 0 ? forced : (long_range ? 0 : (small_gr ? 1 : 2));
  if (var == 1 && !small_gr) var = 2;
  if (big_gr) var = 3;
  const int64_t cols = (int64_t)a.H * a.d;
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  int32_t* tbase = reinterpret_cast<int32_t*>(wsb + band_bytes);
  int32_t* gtbase = tbase + a.nseq + 1;
  int32_t* tseq = gtbase + a.nseq + 1;
  int32_t* gtseq = tseq + tc_max_tiles(a.nseq, a.T);
  __nv_bfloat16* compact = reinterpret_cast<__nv_bfloat16*>(wsb + band_bytes + tc_prefix_bytes(a.nseq, a.T));
  const int64_t cld = 3 * cols;  // compact row stride (elements)
  auto build_maps = [&](CUtensorMap* maps, int v, bool global_rows) {
    const int bn = (v == 0 || v == 3) ? 64 : 32, gr = v == 1 ? 16 : (v == 3 ? 64 : 32);
    const int crow = cap > 0 ? cap : 1;
    const int dd = a.d, H = a.H;
    bool ok = global_rows ? make_map_heads(&maps[0], compact, dd, H, crow, cld, BM)
                          : make_map_heads(&maps[0], a.q, dd, H, a.T, a.ld, BM);
    ok = ok && make_map_heads(&maps[1], a.k, dd, H, a.T, a.ld, gr) && make_map_heads(&maps[2], a.v, dd, H, a.T, a.ld, gr) &&
         make_map_heads(&maps[3], a.k, dd, H, a.T, a.ld, bn) && make_map_heads(&maps[4], a.v, dd, H, a.T, a.ld, bn);
    ok = ok && make_map_heads(&maps[7], a.q, dd, H, a.T, a.ld, gr);
    if (qds) ok = ok && make_map_heads(&maps[5], compact + cols, dd, H, crow, cld, bn) &&
                  make_map_heads(&maps[6], compact + 2 * cols, dd, H, crow, cld, bn);
    else { maps[5] = maps[3]; maps[6] = maps[4]; }
    return ok;
  };
  auto launch_var = [&](int v, dim3 grid, const CUtensorMap* maps, const Params& p) {
    return v == 0 ? launch_kernel<VLONG>(grid, maps, p, st)
         : v == 1 ? launch_kernel<VMID>(grid, maps, p, st)
         : v == 2 ? launch_kernel<VMID32>(grid, maps, p, st)
                  : launch_kernel<VG64>(grid, maps, p, st);
  };

  if (qds) {
    tile128_prefix_kernel<<<1, 1024, 0, st>>>(a.cu, a.qlen, a.nseq, a.glob_cu, gtbase, gtseq);
    SC_CHECK_LAUNCH("tile128_prefix_kernel");
    if (cap > 0) {
      qds_gather_kernel<<<(cap + 7) / 8, 256, 0, st>>>(a.cu, a.qlen, a.nseq, a.glob_cu, a.glob_pos,
                                                       static_cast<const __nv_bfloat16*>(a.q),
                                                       static_cast<const __nv_bfloat16*>(a.k),
                                                       static_cast<const __nv_bfloat16*>(a.v), a.ld,
                                                       (int)cols, cap, compact, a.status);
      SC_CHECK_LAUNCH("qds_gather_kernel");
    }
  }

  Params p;
  p.nseq = a.nseq; p.H = a.H; p.w = w == SC_LINK_FULL ? -1 : w; p.padding = a.padding;
  p.link_cls = L.w[2][0] == SC_LINK_FULL; p.link_query = L.w[2][1] == SC_LINK_FULL;
  p.c2 = 1.4426950408889634f / a.scale;
  p.cu = a.cu; p.qlen = a.qlen; p.tile_base = tbase; p.tile_seq = tseq;
  p.out = static_cast<__nv_bfloat16*>(a.out); p.ld_out = a.ld_out; p.dout = a.d;
  p.qds = qds ? 1 : 0; p.global_rows = 0;
  p.flags = a.flags; p.glob_cu = a.glob_cu; p.glob_pos = a.glob_pos;
  // head rows folded into the doc-rows pass (records in the band kernel's workspace layout)
  const int fneed = full_rows_needed(L, max_qgroup_len);
  p.fold = 1; p.fneed = fneed; p.fmax = fneed > 0 ? fneed : 1;
  p.fold_skip = getenv("SC_TC_FOLD_SKIP") ? atoi(getenv("SC_TC_FOLD_SKIP")) : 0;
  p.head_fast = getenv("SC_TC_HEAD_FAST") ? atoi(getenv("SC_TC_HEAD_FAST")) : 1;
  p.ntiles_max = (int)((a.T + tile_rows - 1) / tile_rows + a.nseq);
  for (int gsrc = 0; gsrc < 2; ++gsrc) {
    p.hl[gsrc][0] = L.w[gsrc][0] == SC_LINK_FULL;
    p.hl[gsrc][1] = L.w[gsrc][1] == SC_LINK_FULL;
    p.hdoc[gsrc] = L.w[gsrc][2] == SC_LINK_FULL;
  }
  p.tile64 = seq_tile_base; p.partials = static_cast<float*>(ws);
  tile128_prefix_kernel<<<1, 1024, 0, st>>>(a.cu, a.qlen, a.nseq, nullptr, tbase, tseq);
  SC_CHECK_LAUNCH("tile128_prefix_kernel");
  CUtensorMap maps[8];
  if (!build_maps(maps, var, false)) return unsupported("cuTensorMapEncodeTiled failed");
  const unsigned ntile_grid = (unsigned)((a.T + BM - 1) / BM + a.nseq);
  int rc = launch_var(var, p.head_fast ? dim3((unsigned)a.H, ntile_grid) : dim3(ntile_grid, (unsigned)a.H), maps, p);
  if (rc) return rc;
  if (qds && cap > 0) {
    // QDS global doc rows: every key of their sequence (R/attention.py:461-470)
    Params pg = p;
    pg.qds = 0; pg.global_rows = 1; pg.tile_base = gtbase; pg.tile_seq = gtseq; pg.link_cls = pg.link_query = 1; pg.fold = 0;
    const int vg = forced >= 0 ? var : (big_gr ? 3 : 0);
    CUtensorMap gmaps[8];
    if (!build_maps(gmaps, vg, true)) return unsupported("cuTensorMapEncodeTiled failed");
    const unsigned gtile_grid = (unsigned)((cap + BM - 1) / BM + a.nseq);
    rc = launch_var(vg, pg.head_fast ? dim3((unsigned)a.H, gtile_grid) : dim3(gtile_grid, (unsigned)a.H), gmaps, pg);
    if (rc) return rc;
  }
  // Head rows: the doc-rows pass left the split-softmax records; fold them into the
  // rows with a FULL doc link.
  return launch_head_merge(a, seq_tile_base, tile_rows, max_qgroup_len, ws, st);
}

}  // namespace sc
