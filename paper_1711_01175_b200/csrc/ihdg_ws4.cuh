// Warp-specialised iHDG-II sweep, version 4 (2D, experimental, opt-in with
// IHDG_SWEEP_IMPL=ws4): two consumer TEAMS on alternating half tiles.
//
// The logical tile of k_sweep_ws (16 consecutive elements of one layer, the
// unit of the stopping-norm partials) is split into two 8-element sub-tiles;
// sub-tile 2j + h goes to team h.  Each team has one consumer warp per SMSP
// holding the L fragments of row tiles cw, cw + 4, ... in registers (19 row
// tiles: 5/5/5/4 per SMSP), so the DMMA work is balanced over the four FP64
// pipes and the two teams' phases (norm / contraction / epilogue / waits)
// interleave on every SMSP instead of running in one lock-step.
//
//   producer warp  : per sub-tile, metadata + TMA bulk copies of s and u^k
//   prep warps (4) : q of the sub-tile (TraceSnapshot) -> qready; the bulk
//                    store of every sub-tile; the logical-tile partial
//                    (team 0 + team 1, fixed order)
//   consumer teams : DMMA contraction of sub-tile j, DMMA norm of sub-tile j-1
#pragma once

#include "ihdg_ws.cuh"

namespace ihdg {

// DMMA norm (C^T Delta C) over the units u = cw + 4 m of one sub-tile, in
// chunks of CH units (register budget of the 5-row-tile consumer warps)
template <int N1, int M, int E, int NCWT, int UPW, int DUE, int DUC, int CH>
__device__ __forceinline__ double norm_units_chunked(const double* __restrict__ dbuf, int cw, int lane,
                                                     const double (&cfr)[2], const double* comp_w) {
  double acc = 0.0;
#pragma unroll
  for (int m0 = 0; m0 < UPW; m0 += CH) {
    double r0[CH], r1[CH];
#pragma unroll
    for (int mm = 0; mm < CH; ++mm) {
      const int u = cw + (m0 + mm) * NCWT;
      const bool valid = (m0 + mm) < UPW && u < E * M;
      const int uu = valid ? u : 0;
      const int t = uu / M, c = uu - (uu / M) * M;
      const double* base = dbuf + t * DUE + c * DUC;
      r0[mm] = 0.0;
      r1[mm] = 0.0;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int kk = 4 * ks + (lane & 3), nn = lane >> 2;
        const double b = (valid && kk < N1 && nn < N1) ? base[ws_dnode(kk, nn)] : 0.0;
        dmma_8x8x4(r0[mm], r1[mm], cfr[ks], b);
      }
    }
#pragma unroll
    for (int mm = 0; mm < CH; ++mm) {
      const int u = cw + (m0 + mm) * NCWT;
      const bool valid = (m0 + mm) < UPW && u < E * M;
      const int c = (valid ? u : 0) % M;
      double y0 = 0.0, y1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int col = 4 * ks + (lane & 3);
        const int src = (lane & ~3) | (col >> 1);
        const double x0 = __shfl_sync(0xffffffffu, r0[mm], src);
        const double x1 = __shfl_sync(0xffffffffu, r1[mm], src);
        dmma_8x8x4(y0, y1, (col & 1) ? x1 : x0, cfr[ks]);
      }
      const double w = valid ? comp_w[c] : 0.0;
      acc = fma(w * y0, y0, acc);
      acc = fma(w * y1, y1, acc);
    }
  }
  return acc;
}

template <int N1, int M, int NCF, int NWC, int NS>
struct W4Cfg {
  static constexpr int D = 2;
  static constexpr int E = 8;                         // sub-tile (DMMA n)
  static constexpr int EL = 16;                       // logical tile (partials)
  static constexpr int NP = N1 * N1;
  static constexpr int NV = M * NP;
  static constexpr int NF = N1;
  static constexpr int KC = NCF * NF;
  static constexpr int NRT = (NV + 7) / 8;
  static constexpr int KS = KC / 4;
  static constexpr int NCWT = 4;                      // consumer warps per team (one per SMSP)
  static constexpr int NCW = 2 * NCWT;
  static constexpr int RTW = (NRT + NCWT - 1) / NCWT;
  static constexpr int UPW = (E * M + NCWT - 1) / NCWT;
  static constexpr int NQW = 4;
  static constexpr int NT = 32 * (NCW + NQW + 1);
  static constexpr int TILE = E * NV;
  static constexpr int QT = E * KC;
  static constexpr int STAGE = 2 * TILE + QT;
  static constexpr int OFF_OUT = NS * STAGE;          // 4 out buffers: team h, parity
  static constexpr int DUC = 8 * N1 + 3;
  static constexpr int DUE = M * DUC;
  static constexpr int DT = E * DUE;
  static constexpr int OFF_D = OFF_OUT + 4 * TILE;    // delta: team h, 2 slots
  static constexpr int NRS = 4;                       // partial slots per team (logical tiles)
  static constexpr int OFF_RED = OFF_D + 4 * DT;
  static constexpr int N_DBL = OFF_RED + 2 * NRS * NCWT;
  static constexpr int NBAR = 3 * NS + 4 + 4;         // full/qready/empty, done[2][2], outfree[4]
  static constexpr size_t BYTES = (size_t)N_DBL * sizeof(double) + NBAR * sizeof(uint64_t);
  static_assert(KC % 4 == 0 && N1 <= 8, "ws4 config");
  static_assert((TILE * sizeof(double)) % 16 == 0, "tile bytes must be 16-byte multiples");
  static_assert(E % NQW == 0, "prep warps split the sub-tile");
  static_assert(BYTES <= 227 * 1024, "shared memory");
};

template <int N1, int M, int NCF, int NWC, int NS>
__global__ void __launch_bounds__(W4Cfg<N1, M, NCF, NWC, NS>::NT, 1)
    k_sweep_ws4(const __grid_constant__ ihdg_sweep_args a) {
  using C = W4Cfg<N1, M, NCF, NWC, NS>;
  constexpr int D = 2, NP = C::NP, NV = C::NV, NF = C::NF, NFACE = 4, KC = C::KC, E = C::E, EL = C::EL;
  constexpr int NRT = C::NRT, KS = C::KS, NCWT = C::NCWT, NCW = C::NCW, RTW = C::RTW, UPW = C::UPW;
  constexpr int NQW = C::NQW, TILE = C::TILE, NRS = C::NRS;

  extern __shared__ __align__(16) double sm[];
  double* out_s = sm + C::OFF_OUT;
  double* d_s = sm + C::OFF_D;
  double* red_s = sm + C::OFF_RED;     // [team][NRS][NCWT]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::N_DBL);
  uint64_t* full_bar = bars;             // [NS] producer -> prep
  uint64_t* qready_bar = bars + NS;      // [NS] prep -> team
  uint64_t* empty_bar = bars + 2 * NS;   // [NS] team -> producer
  uint64_t* done_bar = bars + 3 * NS;    // [2 teams][2] team -> prep, team
  uint64_t* outfree_bar = done_bar + 4;  // [4 out buffers] prep -> team

  __shared__ int cf_s[NCF];
  __shared__ int wc_s[NCF][NWC];
  __shared__ double ww_s[NCF][NWC];
  __shared__ double chol_s[N1 * N1];
  __shared__ int qf_s[KC];
  __shared__ int qt_s[KC][NWC];
  __shared__ long long me0_s[NS];
  __shared__ int mnt_s[NS], mfast_s[NS];
  __shared__ unsigned mcset_s[NS];
  __shared__ int mmask_s[NS][E], mcls_s[NS][E];
  __shared__ int com_s[64];
  __shared__ int last_s;

  ihdg_iter_state* st = a.state;
  if (st->status != IHDG_RUNNING) return;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  Geo geo;
  geo.init(a.g, EL);
  const int64_t ls = geo.ls;
  const double* __restrict__ uo = a.u_old + ls * NV;
  double* __restrict__ un = a.u_new + ls * NV;

  for (int i = tid; i < N1 * N1; i += blockDim.x) chol_s[i] = a.chol1d[i];
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
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&qready_bar[s], NQW);
      mbar_init(&empty_bar[s], NCWT);
    }
    for (int b = 0; b < 4; ++b) {
      mbar_init(&done_bar[b], NCWT);
      mbar_init(&outfree_bar[b], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int fast_class = a.class_of_mask[0];
  const int ntiles = (int)geo.ntiles;
  int n_my = 0;  // logical tiles of this CTA
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) ++n_my;
  const int n_sub = 2 * n_my;
  const int c0 = (int)a.g.cells[0];
  const int per0 = a.g.periodic[0];
  const int nlay = (int)(a.g.layer_end - a.g.layer_begin);
  const int lsi = (int)ls;
  // sub-tile it -> out buffer (team, parity of the team's sub-tile index)
  auto obuf = [](int it) { return (it & 1) * 2 + ((it >> 1) & 1); };

  if (warp == NCW + NQW) {
    // ============================ producer warp ============================
    for (int it = 0; it < n_sub; ++it) {
      const int h = it & 1;
      const int tile = blockIdx.x + (it >> 1) * gridDim.x;
      const int stage = it % NS;
      if (it >= NS) mbar_wait(&empty_bar[stage], ((it / NS) - 1) & 1);
      double* sst = sm + stage * C::STAGE;
      double* ust = sst + TILE;
      STile<D> ti;
      ti.init(a.g, tile, EL, nlay, lsi);
      const int e0 = ti.e0 + h * E;
      int cls = -1;
      if (lane < E) {
        const int mask = ti.mask(h * E + lane, c0, per0);
        cls = com_s[mask];
        mmask_s[stage][lane] = mask;
        mcls_s[stage][lane] = cls;
      }
      const int fast = __all_sync(0xffffffffu, lane >= E || cls == fast_class);
      unsigned cset = (lane < E && cls >= 0 && cls < 32) ? (1u << cls) : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cset |= __shfl_xor_sync(0xffffffffu, cset, o);
      if (lane == 0) {
        me0_s[stage] = e0;
        mnt_s[stage] = E;
        mfast_s[stage] = fast;
        mcset_s[stage] = cset;
      }
      __syncwarp();
      if (lane == 0) {
        const uint32_t bytes = (uint32_t)(E * NV * sizeof(double));
        mbar_arrive_expect_tx(&full_bar[stage], 2 * bytes);
        bulk_g2s(sst, a.s + (int64_t)e0 * NV, bytes, &full_bar[stage]);
        bulk_g2s(ust, uo + (int64_t)e0 * NV, bytes, &full_bar[stage]);
      }
    }
  } else if (warp >= NCW) {
    // ============================ prep warps ===============================
    const int pw = warp - NCW;
    constexpr int HALF = E / NQW;
    constexpr int QM = (HALF * KC + 31) / 32;
    double gv[QM][NWC], gvn[QM][NWC];
    int qs = 0, ql = 0, qsn = 0, qln = 0;
    auto gather = [&](int itg, double (&dst)[QM][NWC], int& in_bits, int& ld_bits) {
      in_bits = 0;
      ld_bits = 0;
      if (itg >= n_sub) return;
      const int h = itg & 1;
      STile<D> tg;
      tg.init(a.g, (int)blockIdx.x + (itg >> 1) * (int)gridDim.x, EL, nlay, lsi);
#pragma unroll
      for (int m = 0; m < QM; ++m) {
        const int idx = lane + 32 * m;
#pragma unroll
        for (int j = 0; j < NWC; ++j) dst[m][j] = 0.0;
        if (idx < HALF * KC) {
          const int t = pw * HALF + idx / KC, k = idx - (idx / KC) * KC;
          const int tl = h * E + t;    // element inside the logical tile
          const int f = qf_s[k];
          if (!(tg.mask(tl, c0, per0) & (1 << f))) {
            const bool in_tile = (f >> 1) == 0 && !((f == 0 && t == 0) || (f == 1 && t == E - 1));
            if (in_tile) {
              in_bits |= 1 << m;
            } else {
              ld_bits |= 1 << m;
              int nb;
              if (f >= 2) {
                nb = tg.e0 + tl + tg.face_off(f);
              } else {
                const int i = tg.i0 + tl;
                nb = tg.e0 + tl + ((f == 0) ? (i > 0 ? -1 : c0 - 1) : (i < c0 - 1 ? 1 : -(c0 - 1)));
              }
              const double* src = uo + (int64_t)nb * NV;
#pragma unroll
              for (int j = 0; j < NWC; ++j) dst[m][j] = __ldg(src + qt_s[k][j]);
            }
          }
        }
      }
    };
    int e0_hist[4] = {0, 0, 0, 0};   // sub-tile it & 3 -> first element
    gather(0, gv, qs, ql);
    for (int it = 0; it < n_sub; ++it) {
      const int stage = it % NS;
      gather(it + 1, gvn, qsn, qln);
      mbar_wait(&full_bar[stage], (it / NS) & 1);
      e0_hist[it & 3] = (int)me0_s[stage];
      const double* sst = sm + stage * C::STAGE;
      const double* ust = sst + TILE;
      double* qst = const_cast<double*>(ust) + TILE;
#pragma unroll
      for (int m = 0; m < QM; ++m) {
        const int idx = lane + 32 * m;
        if (idx < HALF * KC) {
          const int t = pw * HALF + idx / KC, k = idx - (idx / KC) * KC;
          const int ci = k / NF;
          double v = 0.0;
          if (qs & (1 << m)) {
            const int f = qf_s[k];
            const double* src = ust + (t + (f == 0 ? -1 : 1)) * NV;
#pragma unroll
            for (int j = 0; j < NWC; ++j) v = fma(ww_s[ci][j], src[qt_s[k][j]], v);
          } else if (ql & (1 << m)) {
#pragma unroll
            for (int j = 0; j < NWC; ++j) v = fma(ww_s[ci][j], gv[m][j], v);
          }
          qst[ws_qcol<1>(t) * KC + k] = v;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&qready_bar[stage]);
      if (it >= 2) {
        // sub-tile it-2 (same team) is complete: store it
        const int sp = it - 2, h = sp & 1, j = sp >> 1;
        mbar_wait(&done_bar[h * 2 + (j & 1)], (j >> 1) & 1);
        if (pw == 0 && lane == 0) {
          bulk_s2g(un + (int64_t)e0_hist[sp & 3] * NV, out_s + obuf(sp) * TILE, (uint32_t)(E * NV * sizeof(double)));
          bulk_commit();
          // the store of sub-tile it-3 has read its buffer: sub-tile it+1 may reuse it
          if (it >= 3) {
            bulk_wait_read<1>();
            mbar_arrive(&outfree_bar[obuf(it - 3)]);
          }
          // logical tile L: both halves' norms are in once team 1 has
          // finished its sub-tile j = L + 1 (norm of L runs in iteration L + 1)
          if (h == 1 && j >= 1) {
            const int L = j - 1;
            double s = 0.0;
            for (int w = 0; w < NCWT; ++w) s += red_s[(0 * NRS + L % NRS) * NCWT + w];
            for (int w = 0; w < NCWT; ++w) s += red_s[(1 * NRS + L % NRS) * NCWT + w];
            a.tile_partials[blockIdx.x + L * gridDim.x] = a.jac * s;
          }
        }
      }
#pragma unroll
      for (int m = 0; m < QM; ++m)
#pragma unroll
        for (int j = 0; j < NWC; ++j) gv[m][j] = gvn[m][j];
      qs = qsn;
      ql = qln;
    }
    // drain: the last two sub-tiles
    for (int sp = n_sub - 2 > 0 ? n_sub - 2 : 0; sp < n_sub; ++sp) {
      const int h = sp & 1, j = sp >> 1;
      mbar_wait(&done_bar[h * 2 + (j & 1)], (j >> 1) & 1);
      if (pw == 0 && lane == 0) {
        bulk_s2g(un + (int64_t)e0_hist[sp & 3] * NV, out_s + obuf(sp) * TILE, (uint32_t)(E * NV * sizeof(double)));
        bulk_commit();
        if (h == 1 && j >= 1) {
          const int L = j - 1;
          double s = 0.0;
          for (int w = 0; w < NCWT; ++w) s += red_s[(0 * NRS + L % NRS) * NCWT + w];
          for (int w = 0; w < NCWT; ++w) s += red_s[(1 * NRS + L % NRS) * NCWT + w];
          a.tile_partials[blockIdx.x + L * gridDim.x] = a.jac * s;
        }
      }
    }
    if (pw == 0 && lane == 0) bulk_wait<0>();
  } else {
    // ============================ consumer teams ===========================
    const int team = warp / NCWT, cw = warp % NCWT;
    double Lf[RTW][KS];
#pragma unroll
    for (int j = 0; j < RTW; ++j) {
      const int row = (cw + j * NCWT) * 8 + (lane >> 2);
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int k = 4 * ks + (lane & 3);
        const int col = cf_s[k / NF] * NF + (k % NF);
        Lf[j][ks] = (row < NV) ? __ldg(a.LT + ((size_t)fast_class * (NFACE * NF) + col) * NV + row) : 0.0;
      }
    }
    double cfr[2];
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int kk = 4 * ks + (lane & 3), nn = lane >> 2;
      cfr[ks] = (kk < N1 && nn < N1) ? chol_s[kk * N1 + nn] : 0.0;
    }
    double* dteam = d_s + team * 2 * C::DT;
    double* rteam = red_s + team * NRS * NCWT;
    const int n_team = (n_sub - team + 1) / 2;   // sub-tiles team, team + 2, ...
    for (int j = 0; j < n_team; ++j) {
      const int it = 2 * j + team;
      const int stage = it % NS;
      mbar_wait(&qready_bar[stage], (it / NS) & 1);
      const int fast = mfast_s[stage];
      const double* sst = sm + stage * C::STAGE;
      const double* ust = sst + TILE;
      const double* qst = ust + TILE;
      double nsum = 0.0;
      if (j >= 1) {   // norm of the team's previous sub-tile
        mbar_wait(&done_bar[team * 2 + ((j - 1) & 1)], ((j - 1) >> 1) & 1);
        nsum = norm_units_chunked<N1, M, E, NCWT, UPW, C::DUE, C::DUC, 2>(dteam + ((j - 1) & 1) * C::DT, cw, lane,
                                                                          cfr, a.comp_w);
      }
      double acc[RTW][2];
      const int te = 2 * (lane & 3);
#pragma unroll
      for (int j2 = 0; j2 < RTW; ++j2) {
        const int row = (cw + j2 * NCWT) * 8 + (lane >> 2);
        const bool ok = row < NV && (cw + j2 * NCWT) < NRT;
        acc[j2][0] = ok ? sst[te * NV + row] : 0.0;
        acc[j2][1] = ok ? sst[(te + 1) * NV + row] : 0.0;
      }
      const double* qb = qst + (lane >> 2) * KC + (lane & 3);
      if (fast) {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const double b = qb[4 * ks];
#pragma unroll
          for (int j2 = 0; j2 < RTW; ++j2) dmma_8x8x4(acc[j2][0], acc[j2][1], Lf[j2][ks], b);
        }
      } else {
        const unsigned cset = mcset_s[stage];
        for (unsigned rem = cset; rem != 0u; rem &= rem - 1u) {
          const int c = __ffs(rem) - 1;
          for (int ks = 0; ks < KS; ++ks) {
            const int k = 4 * ks + (lane & 3);
            const int col = cf_s[k / NF] * NF + (k % NF);
            const int n = lane >> 2;
            const double b = (mcls_s[stage][ws_elem<1>(n >> 1, 0, n & 1)] == c) ? qb[4 * ks] : 0.0;
#pragma unroll
            for (int j2 = 0; j2 < RTW; ++j2) {
              const int row = (cw + j2 * NCWT) * 8 + (lane >> 2);
              const double av = (row < NV) ? __ldg(a.LT + ((size_t)c * (NFACE * NF) + col) * NV + row) : 0.0;
              dmma_8x8x4(acc[j2][0], acc[j2][1], av, b);
            }
          }
        }
      }
      if (it >= 4) mbar_wait(&outfree_bar[obuf(it)], ((it >> 2) - 1) & 1);
      double* outb = out_s + obuf(it) * TILE;
      double* dcur = dteam + (j & 1) * C::DT;
#pragma unroll
      for (int j2 = 0; j2 < RTW; ++j2) {
        const int row = (cw + j2 * NCWT) * 8 + (lane >> 2);
        if (row < NV && (cw + j2 * NCWT) < NRT) {
          const int r = row, c = r / NP, node = r - c * NP;
          const int doff = c * C::DUC + ws_dnode(node / N1, node - (node / N1) * N1);
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int t = te + v;
            outb[t * NV + row] = acc[j2][v];
            dcur[t * C::DUE + doff] = acc[j2][v] - ust[t * NV + row];
          }
        }
      }
      if (j >= 1) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, o);
        if (lane == 0) rteam[((j - 1) % NRS) * NCWT + cw] = nsum;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty_bar[stage]);
        mbar_arrive(&done_bar[team * 2 + (j & 1)]);
      }
    }
    // drain: norm of the team's last sub-tile
    if (n_team >= 1) {
      const int j = n_team - 1;
      mbar_wait(&done_bar[team * 2 + (j & 1)], (j >> 1) & 1);
      double nsum = norm_units_chunked<N1, M, E, NCWT, UPW, C::DUE, C::DUC, 2>(dteam + (j & 1) * C::DT, cw, lane,
                                                                               cfr, a.comp_w);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, o);
      if (lane == 0) rteam[(j % NRS) * NCWT + cw] = nsum;
    }
  }

  __syncthreads();
  if (tid == 0 && n_my >= 1) {
    // the last logical tile (its team-1 norm ran in the drain)
    const int L = n_my - 1;
    double s = 0.0;
    for (int w = 0; w < NCWT; ++w) s += red_s[(0 * NRS + L % NRS) * NCWT + w];
    for (int w = 0; w < NCWT; ++w) s += red_s[(1 * NRS + L % NRS) * NCWT + w];
    a.tile_partials[blockIdx.x + L * gridDim.x] = a.jac * s;
  }
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
      finalize_block(a.tile_partials, geo.ntiles, st, a.norm_hist);
    }
  }
}

}  // namespace ihdg
