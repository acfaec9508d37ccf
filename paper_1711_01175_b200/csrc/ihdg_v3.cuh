// iHDG-II sweep, version 3: one consumer warp owns one 8-element tile end to
// end, so consumer warps never wait on each other (production path for the
// 2D and 3D BASELINE configs 2-5).
//
//   producer warp  : per tile, metadata + one TMA bulk copy (cp.async.bulk) of
//                    the u^k tile + cp.async gathers of the out-of-tile
//                    neighbour face nodes into an NS-deep stage ring (-> full);
//                    retires stages in order (waits done) and reduces the tile
//                    partials of the stopping norm in a fixed order.
//   prep warps (2) : neighbour face scalars q (TraceSnapshot of iterate k)
//                    for the stage (-> qready).
//   consumer warps : issue the loads of s straight into the DMMA
//                    accumulators (before waiting on the stage), run
//                    u^{k+1} = s + L q on the fp64 tensor core
//                    (mma.sync.m8n8k4.f64; L fragments in shared memory,
//                    conflict-free), store u^{k+1} from registers, write
//                    delta = u^{k+1} - u^k in place over the staged u^k tile
//                    and reduce J |(C^T x .. x C^T) delta|^2 with exact
//                    triangular DFMA passes (warp-local)   (-> done).
//
// HBM per element-DOF: s (LDG), u^k (TMA), u^{k+1} (STG) = 24 B.
#pragma once

#include "ihdg_stream.cuh"

namespace ihdg {

template <int D, int N1, int M, int NCF, int NWC, int NS, int NCW, int PF, int NQW_ = 2>
struct V3Cfg {
  static constexpr int E = 8;                     // elements per physical tile (DMMA n)
  static constexpr int NP = Pow<N1, D>::v;
  static constexpr int NV = M * NP;
  static constexpr int NF = Pow<N1, D - 1>::v;
  static constexpr int NFACE = 2 * D;
  static constexpr int KC = NCF * NF;
  static constexpr int NRT = (NV + 7) / 8;        // DMMA row tiles
  static constexpr int KS = KC / 4;               // DMMA k steps
  static constexpr int NQW = NQW_;                // prep warps
  static constexpr int NT = 32 * (NCW + NQW + 1);
  // registers: the file is split over 4 SMSPs, so the cap follows the busiest SMSP
  static constexpr int WPS = (NT / 32 + 3) / 4;   // warps per SMSP
  static constexpr int MAXREG = (16384 / (32 * WPS)) / 8 * 8 > 255 ? 255 : (16384 / (32 * WPS)) / 8 * 8;
  // register prefetch of the next tile's s only when one warp per SMSP cannot
  // be covered by another consumer warp
  static constexpr bool PREF = WPS <= 2 && NCW <= 4;
  // shared-memory strides, chosen bank-conflict-free (64-bit accesses, one
  // wavefront per half-warp): the staged u^k tile is copied per element into
  // an element stride ES with 2 ES = 4 (mod 16) double-banks when NV is even
  // (one 16-byte-aligned bulk copy per element); q rows use KCP = 4 (mod 8).
  static constexpr int ES = (NV % 2 == 0) ? NV + ((2 - NV % 8 + 8) % 8) : NV;
  static constexpr int KCP = KC + ((4 - KC % 8 + 8) % 8);
  static constexpr bool TFAST = ES != NV;   // norm lines: element index fastest
  static constexpr int TILE = E * ES;
  static constexpr int HALO = 0;                  // out-of-tile faces: prep warps load them directly
  static constexpr int QT = E * KCP;
  static constexpr int STAGE = TILE + HALO + QT;  // doubles
  static constexpr int LFR = NRT * KS * 32;       // L fragments (doubles)
  static constexpr int OFF_L = NS * STAGE;
  static constexpr int N_DBL = OFF_L + LFR;
  static constexpr size_t BYTES = (size_t)N_DBL * sizeof(double) + 3 * NS * sizeof(uint64_t);
  static constexpr int LPL = NP / N1;             // norm lines per (element, component) and axis
  static constexpr int NLINES = E * M * LPL;
  static_assert(KC % 4 == 0, "DMMA k");
  static_assert(E % 2 == 0 && (E * NV * sizeof(double)) % 16 == 0, "bulk copy alignment");
  static_assert(ES == NV || ((NV * sizeof(double)) % 16 == 0 && (ES * sizeof(double)) % 16 == 0),
                "per-element bulk copies need 16-byte sizes and strides");
  static_assert(E % NQW == 0, "prep split");
};

template <int D, int N1, int M, int NCF, int NWC, int NS, int NCW, int PF, int NQW_>
__global__ void __launch_bounds__(V3Cfg<D, N1, M, NCF, NWC, NS, NCW, PF, NQW_>::NT, 1) __maxnreg__((V3Cfg<D, N1, M, NCF, NWC, NS, NCW, PF, NQW_>::MAXREG))
    k_sweep_v3(const ihdg_sweep_args a) {
  using C = V3Cfg<D, N1, M, NCF, NWC, NS, NCW, PF, NQW_>;
  constexpr int E = C::E, NP = C::NP, NV = C::NV, NF = C::NF, NFACE = C::NFACE, KC = C::KC;
  constexpr int NRT = C::NRT, KS = C::KS, NQW = C::NQW, TILE = C::TILE;

  extern __shared__ __align__(16) double sm[];
  const double* lfr_s = sm + C::OFF_L;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::N_DBL);
  uint64_t* full_bar = bars;
  uint64_t* qready_bar = bars + NS;
  uint64_t* done_bar = bars + 2 * NS;

  __shared__ int fv_s[NFACE][NF];
  __shared__ int cf_s[NCF];
  __shared__ int wc_s[NCF][NWC];
  __shared__ double ww_s[NCF][NWC];
  __shared__ double chol_s[N1 * N1];
  __shared__ double cw_s[IHDG_MAX_COMP];
  __shared__ int qf_s[KC], qh_s[KC];
  __shared__ int qt_s[KC][NWC];
  __shared__ int mfast_s[NS];
  // item ids of the stage's current load / q (phase-aliasing guard: a warp
  // that waits on stage s for item it first sees it published, so the
  // barrier is at most one phase behind its parity wait)
  __shared__ int mload_s[NS], mq_s[NS];
  __shared__ unsigned mcset_s[NS];
  __shared__ int mcls_s[NS][E];
  __shared__ double part_s[NS];
  __shared__ int com_s[64];                 // class_of_mask
  __shared__ int last_s;

  ihdg_iter_state* st = a.state;
  pdl_launch_dependents();   // the next launch may start its own prologue
  V3_DECL

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  Geo geo;
  geo.init(a.g, E * PF);  // logical tile = PF physical tiles = the generic kernel's tile
  const int64_t ls = geo.ls;
  const double* __restrict__ uo = a.u_old + ls * NV;
  double* __restrict__ un = a.u_new + ls * NV;
  const int fast_class = a.class_of_mask[0];

  for (int i = tid; i < NFACE * NF; i += blockDim.x) fv_s[i / NF][i % NF] = face_node_vidx(D, N1, i / NF, i % NF);
  for (int i = tid; i < N1 * N1; i += blockDim.x) chol_s[i] = a.chol1d[i];
  if (tid < IHDG_MAX_COMP) cw_s[tid] = a.comp_w[tid];
  if (tid < 64) com_s[tid] = a.class_of_mask[tid];
  if (tid == 0) {
    int n = 0;
    for (int f = 0; f < NFACE && n < NCF; ++f) {
      if (!a.coupled[f]) continue;
      cf_s[n] = f;
      int j = 0;
      for (int c = 0; c < M && j < NWC; ++c)
        if (a.face_w[f][c] != 0.0) {
          wc_s[n][j] = c;
          ww_s[n][j] = a.face_w[f][c];
          ++j;
        }
      for (; j < NWC; ++j) {
        wc_s[n][j] = 0;
        ww_s[n][j] = 0.0;
      }
      ++n;
    }
    for (int k = 0; k < KC; ++k) {
      const int ci = k / NF, nn = k % NF, f = cf_s[ci];
      qf_s[k] = f;
      for (int j = 0; j < NWC; ++j) qt_s[k][j] = wc_s[ci][j] * NP + face_node_vidx(D, N1, f ^ 1, nn);
      qh_s[k] = ci * NWC * NF + nn;
    }
    for (int s = 0; s < NS; ++s) {
      mload_s[s] = -1;
      mq_s[s] = -1;
      mbar_init(&full_bar[s], 1);
      mbar_init(&qready_bar[s], 1);
      mbar_init(&done_bar[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // interior-class L in DMMA A-fragment order: frag (rt, ks), lane l ->
  // L[8 rt + (l>>2)][4 ks + (l&3)]; one 256-byte contiguous run per fragment
  for (int idx = tid; idx < C::LFR; idx += blockDim.x) {
    const int l = idx & 31, fr = idx >> 5;
    const int rt = fr / KS, ks = fr - (fr / KS) * KS;
    const int row = rt * 8 + (l >> 2);
    const int k = 4 * ks + (l & 3);
    const int col = cf_s[k / NF] * NF + (k % NF);
    sm[C::OFF_L + idx] = (row < NV) ? a.LT[((size_t)fast_class * (NFACE * NF) + col) * NV + row] : 0.0;
  }
  __syncthreads();
  // everything above reads only launch-invariant data (operators, tables);
  // the iterate, s and the iteration state belong to the previous launches
  pdl_wait();
  if (st->status != IHDG_RUNNING) return;

  V3_T0(tk0);
  const int nlog = (int)geo.ntiles;
  const int n_log_my = nlog > (int)blockIdx.x ? (nlog - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int n_items = n_log_my * PF;
  const int nlay = (int)(a.g.layer_end - a.g.layer_begin);
  const int lsi = (int)ls;
  auto phys_of = [&](int it) { return ((int)blockIdx.x + (it / PF) * (int)gridDim.x) * PF + it % PF; };

  if (warp == NCW + NQW) {
    // ============================ producer warp ============================
    // retires stages in order (tile partials in a fixed order) and issues one
    // TMA bulk copy of the u^k tile per stage
    double pacc = 0.0;
    auto retire = [&](int j) {
      const int sj = j % NS;
      V3_T0(tr);
      mbar_wait(&done_bar[sj], (j / NS) & 1);
      V3_ACC(0, tr);
      pacc += part_s[sj];
      if (j % PF == PF - 1) {
        if (lane == 0) a.tile_partials[(int)blockIdx.x + (j / PF) * (int)gridDim.x] = a.jac * pacc;
        pacc = 0.0;
      }
    };
    for (int it = 0; it < n_items; ++it) {
      const int stage = it % NS;
      if (it >= NS) retire(it - NS);
      V3_T0(tl);
      if (lane == 0) {
        STile<D> ti;
        ti.e0 = phys_of(it) * E;   // tiles are E consecutive elements of a row, c0 % E == 0
        constexpr uint32_t bytes = (uint32_t)(E * NV * sizeof(double));
        *(volatile int*)&mload_s[stage] = it;   // stage free: item it - NS retired
        mbar_arrive_expect_tx(&full_bar[stage], bytes);
        if constexpr (C::ES == NV) {
          bulk_g2s(sm + stage * C::STAGE, uo + (int64_t)ti.e0 * NV, bytes, &full_bar[stage]);
        } else {
#pragma unroll
          for (int t = 0; t < E; ++t)
            bulk_g2s(sm + stage * C::STAGE + t * C::ES, uo + (int64_t)(ti.e0 + t) * NV,
                     (uint32_t)(NV * sizeof(double)), &full_bar[stage]);
        }
      }
      __syncwarp();
      V3_ACC(9, tl);
    }
    for (int j = n_items > NS ? n_items - NS : 0; j < n_items; ++j) retire(j);
  } else if (warp >= NCW) {
    // ============================ prep warps ===============================
    // prep warp pw owns items pw, pw + NQW, ...: tile metadata + neighbour
    // face scalars q (TraceSnapshot of iterate k).  Out-of-tile neighbour face
    // nodes of its NEXT item are loaded from global (L2) into registers while
    // the current item is processed.
    const int pw = warp - NCW;
    const int c0 = (int)a.g.cells[0];
    const int per0 = a.g.periodic[0];
    constexpr int QM = (E * KC + 31) / 32;
    // per-lane entry constants, hoisted out of the item loop: entry m of this
    // lane is (element t, column k) with k's face f and its gather offsets /
    // weights (TraceSnapshot layout, fixed for the launch)
    int ent_t[QM], ent_f[QM], ent_q[QM][NWC];
#pragma unroll
    for (int m = 0; m < QM; ++m) {
      const int idx = lane + 32 * m;
      const int t = idx < E * KC ? idx / KC : 0, k = idx < E * KC ? idx - (idx / KC) * KC : 0;
      ent_t[m] = idx < E * KC ? t : -1;
      ent_f[m] = qf_s[k];
#pragma unroll
      for (int j = 0; j < NWC; ++j) ent_q[m][j] = qt_s[k][j];
    }
    double gv[QM][NWC], gvn[QM][NWC];
    int qsn = 0;      // bit m: entry m of the next item is an in-tile neighbour
    int qln = 0;      // bit m: entry m of the next item was loaded from global
    int qs = 0, ql = 0;
    STile<D> tnext;
    auto gather = [&](int itg, double (&dst)[QM][NWC], int& in_tile_bits, int& load_bits) {
      in_tile_bits = 0;
      load_bits = 0;
      if (itg >= n_items) return;
      STile<D>& tg = tnext;
      tg.init(a.g, phys_of(itg), E, nlay, lsi);
      // missing neighbours: faces of axes >= 1 are tile-uniform, x faces only
      // at the tile ends
      int hm = 0;
#pragma unroll
      for (int f = 2; f < NFACE; ++f)
        if (!tg.has[f]) hm |= 1 << f;
      const bool xlo = !per0 && tg.i0 == 0, xhi = !per0 && tg.i0 + E == c0;
#pragma unroll
      for (int m = 0; m < QM; ++m) {
#pragma unroll
        for (int j = 0; j < NWC; ++j) dst[m][j] = 0.0;
        const int t = ent_t[m], f = ent_f[m];
        if (t >= 0) {
          const bool miss = f >= 2 ? ((hm >> f) & 1) : (f == 0 ? (t == 0 && xlo) : (t == E - 1 && xhi));
          if (!miss) {
            const bool in_tile = (f >> 1) == 0 && !((f == 0 && t == 0) || (f == 1 && t == E - 1));
            if (in_tile) {
              in_tile_bits |= 1 << m;
            } else {
              load_bits |= 1 << m;
              int nb;
              if (f >= 2) {
                nb = tg.e0 + t + tg.face_off(f);
              } else {
                const int i = tg.i0 + t;
                nb = tg.e0 + t + ((f == 0) ? (i > 0 ? -1 : c0 - 1) : (i < c0 - 1 ? 1 : -(c0 - 1)));
              }
              const double* src = uo + (int64_t)nb * NV;
#pragma unroll
              for (int j = 0; j < NWC; ++j) dst[m][j] = __ldg(src + ent_q[m][j]);
            }
          }
        }
      }
    };
    gather(pw, gv, qs, ql);
    for (int it = pw; it < n_items; it += NQW) {
      const int stage = it % NS;
      const STile<D> ti = tnext;   // geometry of item it (computed by its gather)
      gather(it + NQW, gvn, qsn, qln);
      V3_T0(tp);
      while (*(volatile int*)&mload_s[stage] != it) {
      }
      mbar_wait(&full_bar[stage], (it / NS) & 1);
      V3_ACC(1, tp);
      V3_T0(tq);
      // stage metadata: written only after full (the producer refills a stage
      // after its previous consumer is done with it)
      {
        int cls = -1;
        if (lane < E) {
          cls = com_s[ti.mask(lane, c0, per0)];
          mcls_s[stage][lane] = cls;
        }
        const int fast = __all_sync(0xffffffffu, lane >= E || cls == fast_class);
        unsigned cset = (lane < E && cls >= 0 && cls < 32) ? (1u << cls) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cset |= __shfl_xor_sync(0xffffffffu, cset, o);
        if (lane == 0) {
          mfast_s[stage] = fast;
          mcset_s[stage] = cset;
        }
      }
      const double* ust = sm + stage * C::STAGE;
      double* qst = sm + stage * C::STAGE + TILE;
#pragma unroll
      for (int m = 0; m < QM; ++m) {
        const int t = ent_t[m];
        if (t >= 0) {
          const int k = lane + 32 * m - t * KC;
          const double* w = ww_s[k / NF];
          double v = 0.0;
          if (qs & (1 << m)) {
            const double* src = ust + (t + (ent_f[m] == 0 ? -1 : 1)) * C::ES;
#pragma unroll
            for (int j = 0; j < NWC; ++j) v = fma(w[j], src[ent_q[m][j]], v);
          } else if (ql & (1 << m)) {
#pragma unroll
            for (int j = 0; j < NWC; ++j) v = fma(w[j], gv[m][j], v);
          }
          qst[t * C::KCP + k] = v;
        }
      }
      __syncwarp();
      V3_ACC(2, tq);
      if (lane == 0) {
        *(volatile int*)&mq_s[stage] = it;
        mbar_arrive(&qready_bar[stage]);
      }
#pragma unroll
      for (int m = 0; m < QM; ++m)
#pragma unroll
        for (int j = 0; j < NWC; ++j) gv[m][j] = gvn[m][j];
      qs = qsn;
      ql = qln;
    }
  } else {
    // ============================ consumer warps ===========================
    const int te = 2 * (lane & 3);      // D-fragment columns (elements) of this lane
    const int rsub = lane >> 2;         // D-fragment row inside a row tile
    // s of this warp's first tile -> accumulators; afterwards the s loads of
    // the next tile are issued before the current tile is computed
    double acc[NRT][2], accn[C::PREF ? NRT : 1][2];
    auto load_s = [&](int it_load, double (&dst)[NRT][2]) {
      if (it_load < n_items) {
        const double* sg = a.s + (int64_t)(phys_of(it_load) * E) * NV;
#pragma unroll
        for (int rt = 0; rt < NRT; ++rt) {
          const int row = rt * 8 + rsub;
          dst[rt][0] = (row < NV) ? __ldcs(sg + te * NV + row) : 0.0;
          dst[rt][1] = (row < NV) ? __ldcs(sg + (te + 1) * NV + row) : 0.0;
        }
      }
    };
    if constexpr (C::PREF) load_s(warp, acc);
    for (int it = warp; it < n_items; it += NCW) {
      const int stage = it % NS;
      const int e0 = phys_of(it) * E;
      if constexpr (C::PREF) load_s(it + NCW, *reinterpret_cast<double(*)[NRT][2]>(&accn[0][0]));
      else load_s(it, acc);
      V3_T0(tc);
      while (*(volatile int*)&mq_s[stage] != it) {
      }
      mbar_wait(&qready_bar[stage], (it / NS) & 1);
      V3_ACC(3, tc);
      V3_T0(tm);
      double* ust = sm + stage * C::STAGE;
      const double* qb = ust + TILE + C::HALO + rsub * C::KCP + (lane & 3);
      if (mfast_s[stage]) {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const double b = qb[4 * ks];
#pragma unroll
          for (int rt = 0; rt < NRT; ++rt) dmma_8x8x4(acc[rt][0], acc[rt][1], lfr_s[(rt * KS + ks) * 32 + lane], b);
        }
      } else {
        // one masked pass per operator class present in the tile
        const unsigned cset = mcset_s[stage];
        const int mycls = mcls_s[stage][rsub];
        for (unsigned rem = cset; rem != 0u; rem &= rem - 1u) {
          const int c = __ffs(rem) - 1;
          for (int ks = 0; ks < KS; ++ks) {
            const double b = (mycls == c) ? qb[4 * ks] : 0.0;
            const int k = 4 * ks + (lane & 3);
            const int col = cf_s[k / NF] * NF + (k % NF);
            const double* Lc = a.LT + ((size_t)c * (NFACE * NF) + col) * NV;
#pragma unroll
            for (int rt = 0; rt < NRT; ++rt) {
              const int row = rt * 8 + rsub;
              dmma_8x8x4(acc[rt][0], acc[rt][1], (row < NV) ? __ldg(Lc + row) : 0.0, b);
            }
          }
        }
      }
      V3_ACC(4, tm);
      V3_T0(te2);
      // u^{k+1} -> global (64-byte runs), delta in place over the staged u^k
      double* ug = un + (int64_t)e0 * NV;
#pragma unroll
      for (int rt = 0; rt < NRT; ++rt) {
        const int row = rt * 8 + rsub;
        if (row < NV) {
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int t = te + v;
            __stcs(ug + t * NV + row, acc[rt][v]);
            ust[t * C::ES + row] = acc[rt][v] - ust[t * C::ES + row];
          }
        }
      }
      __syncwarp();
      V3_ACC(5, te2);
      V3_T0(tn);
      // ||delta||_M^2 = J |(C^T x ... x C^T) delta|^2, M1 = C C^T: one exact
      // triangular pass per axis over the lines of the node grid (in place)
      double nsum = 0.0;
      int mul = 1;
#pragma unroll
      for (int ax = 0; ax < D; ++ax) {
        const bool last_ax = ax == D - 1;
#pragma unroll
        for (int m = 0; m < (C::NLINES + 31) / 32; ++m) {
          const int ln = lane + 32 * m;
          if (ln < C::NLINES) {
            int t, c, rem;
            if constexpr (C::TFAST) {
              t = ln % E;
              c = (ln / E) % M;
              rem = ln / (E * M);
            } else {
              t = ln / (M * C::LPL);
              c = (ln / C::LPL) % M;
              rem = ln % C::LPL;
            }
            int base = t * C::ES + c * NP;
            int mb = 1;
#pragma unroll
            for (int b = 0; b < D; ++b) {
              if (b != ax) {
                base += (rem % N1) * mb;
                rem /= N1;
              }
              mb *= N1;
            }
            double x[N1];
#pragma unroll
            for (int i = 0; i < N1; ++i) x[i] = ust[base + i * mul];
            double sq = 0.0;
#pragma unroll
            for (int i = 0; i < N1; ++i) {
              double y = 0.0;
#pragma unroll
              for (int ip = i; ip < N1; ++ip) y = fma(chol_s[ip * N1 + i], x[ip], y);
              if (last_ax) sq = fma(y, y, sq);
              else ust[base + i * mul] = y;
            }
            if (last_ax) nsum = fma(cw_s[c], sq, nsum);
          }
        }
        __syncwarp();
        mul *= N1;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, o);
      V3_ACC(7, tn);
      if (lane == 0) {
        part_s[stage] = nsum;
        mbar_arrive(&done_bar[stage]);  // release: part_s, stage no longer read
      }
      if constexpr (C::PREF) {
#pragma unroll
        for (int rt = 0; rt < NRT; ++rt) {
          acc[rt][0] = accn[rt][0];
          acc[rt][1] = accn[rt][1];
        }
      }
    }
  }

#ifdef IHDG_WS_PROF
  if (tid == 0) V3_ACC(6, tk0);
  V3_FLUSH;
#endif
  if (a.finalize) {
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const unsigned tk = atomicAdd(&st->ticket, 1u);
      last_s = (tk == gridDim.x - 1);
    }
    __syncthreads();
    if (last_s) {
      __threadfence();
      int64_t n_rows, row_len;
      partial_rows(geo, n_rows, row_len);
      finalize_block(a.tile_partials, n_rows, row_len, st, a.norm_hist);
    }
  }
}

}  // namespace ihdg
