// Warp-specialised iHDG-II sweep, version 3 (2D; production path for
// BASELINE config 5).  Same algorithm, tiles and HBM traffic as k_sweep_ws;
// the roles are re-cut so that no role sits on the per-tile critical path
// except the DMMA contraction:
//
//   producer warp   : per tile, metadata + TMA bulk copies of the s and u^k
//                     tiles into an NS-stage ring                -> full[stage]
//   consumer warps  : (8, two per SMSP) neighbour face scalars q
//                     (TraceSnapshot) for the tile -- in-tile
//                     faces from the staged u^k, out-of-tile faces from
//                     registers gathered one tile ahead -- then one named
//                     barrier, DMMA contraction u^{k+1} = s + L q (L fragments
//                     in registers, lifted apply_local),
//                     u^{k+1} and delta = u^{k+1} - u^k to shared memory; an
//                     elected consumer thread issues the bulk store of the
//                     previous tile                   -> empty[stage], dfull[slot]
//   norm warps      : (4, one per SMSP) exact stopping norm of the delta
//                     slot on the DFMA pipe (norm_pass_dfma), fixed-order tile
//                     partial                                   -> dfree[slot]
//
// The prep warps of k_sweep_ws (q + stores) were the measured bottleneck:
// their latency-bound gather/q loop ran ~3.5k cycles per tile on two warps
// while the consumers waited on qready (tools/ws_roles.py).  Spreading q over
// the 256 consumer threads costs each of them 1-2 entries per tile.
#pragma once

#include "ihdg_ws.cuh"

namespace ihdg {

// Exact stopping norm of one pass = 4 (element, component) units on the DFMA
// pipe: ||delta||_M^2 = w_c |C^T Delta C|_F^2 with M1 = C C^T (C lower
// triangular, entries from the kernel parameters -> constant-bank operands).
// Lane (x = lane & 3, j = lane >> 2) owns element t = g + (E/4) x, column j:
//   pass 1: R[:, j] = C^T Delta[:, j]      (column read, written back in place)
//   pass 2: Y[j, :] = R[j, :] C, sum Y^2    (row read)
// 441 FMA per unit for N1 = 7 (the padded 8x8x8 DMMA form spends 1024).  The
// delta tile uses the state layout (element stride NV, node row stride N1):
// with E = 16 the epilogue stores and both passes are bank-conflict free
// (4 lanes x 7 columns / rows per half-warp land on distinct double banks).
template <int N1, int M, int E, int NP, int NV>
__device__ __forceinline__ double norm_pass_dfma(double* __restrict__ dbuf, int pid, int lane,
                                                 const ihdg_sweep_args& a) {
  const int x = lane & 3, j = lane >> 2;
  const int g = pid / M, c = pid - g * M;
  const int t = g + (E / 4) * x;
  const bool act = j < N1;
  const int jj = act ? j : N1 - 1;
  double* base = dbuf + t * NV + c * NP;
  double d[N1], r[N1];
#pragma unroll
  for (int k = 0; k < N1; ++k) d[k] = base[k * N1 + jj];
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    double v = 0.0;
#pragma unroll
    for (int k = i; k < N1; ++k) v = fma(a.chol[k * N1 + i], d[k], v);
    r[i] = v;
  }
  __syncwarp();
  if (act) {
#pragma unroll
    for (int i = 0; i < N1; ++i) base[i * N1 + j] = r[i];
  }
  __syncwarp();
#pragma unroll
  for (int l = 0; l < N1; ++l) d[l] = base[jj * N1 + l];
  double s = 0.0;
#pragma unroll
  for (int l = 0; l < N1; ++l) {
    double y = 0.0;
#pragma unroll
    for (int q = l; q < N1; ++q) y = fma(d[q], a.chol[q * N1 + l], y);
    s = fma(y, y, s);
  }
  return act ? a.comp_w[c] * s : 0.0;
}


template <int N1, int M, int NCF, int NWC, int E, int NS>
struct W3Cfg {
  static constexpr int D = 2;
  static constexpr int NP = N1 * N1;
  static constexpr int NV = M * NP;
  static constexpr int NF = N1;
  static constexpr int KC = NCF * NF;
  static constexpr int NRT = (NV + 7) / 8;
  static constexpr int KS = KC / 4;
  static constexpr int NEG = E / 8;
  static constexpr int NCW = 8;                       // consumer warps (2 per SMSP)
  static constexpr int NNW = 4;                       // norm warps (1 per SMSP)
  static constexpr int NT = 32 * (NCW + NNW + 1);
  static constexpr int RTW = (NRT + NCW - 1) / NCW;
  static constexpr int NPASS = (E / 4) * M;
  static constexpr int TILE = E * NV;
  static constexpr int QE = E * KC;                   // q entries per tile
  static constexpr int QPT = (QE + 32 * NCW - 1) / (32 * NCW);  // entries per consumer thread
  static constexpr int STAGE = 2 * TILE;
  static constexpr int NDB = 2;                       // delta ring (consumers -> norm warps)
  static constexpr int OFF_OUT = NS * STAGE;
  static constexpr int OFF_Q = OFF_OUT + 2 * TILE;    // q double buffer
  static constexpr int OFF_D = OFF_Q + 2 * QE;
  static constexpr int OFF_RED = OFF_D + NDB * TILE;
  static constexpr int N_DBL = OFF_RED + 32 * NDB;
  static constexpr int NBAR = 2 * NS + 2 * NDB;
  static constexpr size_t BYTES = (size_t)N_DBL * sizeof(double) + NBAR * sizeof(uint64_t);
  static_assert(KC % 4 == 0 && E % 8 == 0 && E <= 32 && N1 <= 8, "ws3 config");
  static_assert((TILE * sizeof(double)) % 16 == 0, "tile bytes must be 16-byte multiples");
  static_assert(E % 4 == 0 && N1 * N1 <= IHDG_CHOL_MAX, "norm passes");
  static_assert(BYTES <= 227 * 1024, "shared memory");
};

template <int N1, int M, int NCF, int NWC, int E, int NS>
__global__ void __launch_bounds__(W3Cfg<N1, M, NCF, NWC, E, NS>::NT, 1)
    k_sweep_ws3(const __grid_constant__ ihdg_sweep_args a) {
  using C = W3Cfg<N1, M, NCF, NWC, E, NS>;
  constexpr int D = 2, NP = C::NP, NV = C::NV, NF = C::NF, NFACE = 4, KC = C::KC;
  constexpr int NRT = C::NRT, KS = C::KS, NEG = C::NEG, NCW = C::NCW, RTW = C::RTW;
  constexpr int TILE = C::TILE, NNW = C::NNW, NDB = C::NDB, QE = C::QE, QPT = C::QPT;

  extern __shared__ __align__(16) double sm[];
  double* out_s = sm + C::OFF_OUT;
  double* q_s = sm + C::OFF_Q;
  double* d_s = sm + C::OFF_D;
  double* red_s = sm + C::OFF_RED;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::N_DBL);
  uint64_t* full_bar = bars;              // [NS]  producer -> consumers
  uint64_t* empty_bar = bars + NS;        // [NS]  consumers -> producer
  uint64_t* dfull_bar = bars + 2 * NS;    // [NDB] consumers -> norm warps
  uint64_t* dfree_bar = dfull_bar + NDB;  // [NDB] norm warps -> consumers

  __shared__ int cf_s[NCF];
  __shared__ int wc_s[NCF][NWC];
  __shared__ double ww_s[NCF][NWC];
  __shared__ int qf_s[KC];
  __shared__ int qt_s[KC][NWC];
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
  geo.init(a.g, E);
  const int64_t ls = geo.ls;
  const double* __restrict__ uo = a.u_old + ls * NV;
  double* __restrict__ un = a.u_new + ls * NV;

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
      mbar_init(&empty_bar[s], NCW);
    }
    for (int b = 0; b < NDB; ++b) {
      mbar_init(&dfull_bar[b], NCW);
      mbar_init(&dfree_bar[b], NNW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int fast_class = a.class_of_mask[0];
  const int ntiles = (int)geo.ntiles;
  int n_my = 0;  // tiles of this CTA
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) ++n_my;
  const int c0 = (int)a.g.cells[0];
  const int per0 = a.g.periodic[0];
  const int nlay = (int)(a.g.layer_end - a.g.layer_begin);
  const int lsi = (int)ls;

  if (warp == NCW + NNW) {
    // ============================ producer warp ============================
    for (int it = 0; it < n_my; ++it) {
      const int tile = blockIdx.x + it * gridDim.x;
      const int stage = it % NS;
      if (it >= NS) mbar_wait(&empty_bar[stage], ((it / NS) - 1) & 1);
      double* sst = sm + stage * C::STAGE;
      double* ust = sst + TILE;
      STile<D> ti;
      ti.init(a.g, tile, E, nlay, lsi);
      int cls = -1;
      if (lane < E) {
        const int mask = ti.mask(lane, c0, per0);
        cls = com_s[mask];
        mmask_s[stage][lane] = mask;
        mcls_s[stage][lane] = cls;
      }
      const int fast = __all_sync(0xffffffffu, lane >= E || cls == fast_class);
      unsigned cset = (lane < E && cls >= 0 && cls < 32) ? (1u << cls) : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cset |= __shfl_xor_sync(0xffffffffu, cset, o);
      if (lane == 0) {
        mnt_s[stage] = ti.nt;
        mfast_s[stage] = fast;
        mcset_s[stage] = cset;
      }
      __syncwarp();
      if (lane == 0) {
        const uint32_t bytes = (uint32_t)(ti.nt * NV * sizeof(double));
        mbar_arrive_expect_tx(&full_bar[stage], 2 * bytes);  // release: metadata above
        bulk_g2s(sst, a.s + (int64_t)ti.e0 * NV, bytes, &full_bar[stage]);
        bulk_g2s(ust, uo + (int64_t)ti.e0 * NV, bytes, &full_bar[stage]);
      }
    }
  } else if (warp >= NCW) {
    // ============================ norm warps ===============================
    const int nw = warp - NCW;
    for (int it = 0; it < n_my; ++it) {
      const int slot = it % NDB;
      mbar_wait(&dfull_bar[slot], (it / NDB) & 1);
      double nsum = 0.0;
      for (int pid = nw; pid < C::NPASS; pid += NNW)
        nsum += norm_pass_dfma<N1, M, E, NP, NV>(d_s + slot * TILE, pid, lane, a);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, o);
      if (lane == 0) {
        red_s[slot * 32 + nw] = nsum;
        mbar_arrive(&dfree_bar[slot]);
      }
      named_bar_sync(1, NNW * 32);
      if (nw == 0 && lane == 0) {
        double t = 0.0;
        for (int w = 0; w < NNW; ++w) t += red_s[slot * 32 + w];
        a.tile_partials[blockIdx.x + it * gridDim.x] = a.jac * t;
      }
    }
  } else {
    // ============================ consumer warps ===========================
    const int ctid = tid;  // 0 .. 32 NCW - 1
    double Lf[RTW][KS];
#pragma unroll
    for (int j = 0; j < RTW; ++j) {
      const int row = (warp + j * NCW) * 8 + (lane >> 2);
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int k = 4 * ks + (lane & 3);
        const int col = cf_s[k / NF] * NF + (k % NF);
        Lf[j][ks] = (row < NV) ? __ldg(a.LT + ((size_t)fast_class * (NFACE * NF) + col) * NV + row) : 0.0;
      }
    }
    // this thread's q entries e = ctid + 256 r: element t, entry k, face f,
    // neighbour node offsets, weights; in-tile x faces read the staged u^k
    int et[QPT], ek[QPT], ef[QPT], eoff[QPT][NWC], ein[QPT], eq[QPT];
    double ew[QPT][NWC];
#pragma unroll
    for (int r = 0; r < QPT; ++r) {
      const int e = ctid + 32 * NCW * r;
      const bool v = e < QE;
      const int ee = v ? e : 0;
      et[r] = ee / KC;
      ek[r] = ee - et[r] * KC;
      ef[r] = v ? qf_s[ek[r]] : -1;
      const int ci = ek[r] / NF;
#pragma unroll
      for (int j = 0; j < NWC; ++j) {
        eoff[r][j] = qt_s[ek[r]][j];
        ew[r][j] = ww_s[ci][j];
      }
      const int f = ef[r], t = et[r];
      ein[r] = (f == 0 && t > 0) ? -1 : ((f == 1 && t < E - 1) ? 1 : 0);  // in-tile neighbour (t +- 1)
      eq[r] = ws_qcol<NEG>(t) * KC + ek[r];
    }
    // out-of-tile neighbour face nodes of tile itg -> registers
    double gv[QPT][NWC];
    auto gather = [&](int itg) {
      if (itg >= n_my) return;
      STile<D> tg;
      tg.init(a.g, (int)blockIdx.x + itg * (int)gridDim.x, E, nlay, lsi);
#pragma unroll
      for (int r = 0; r < QPT; ++r) {
        const int f = ef[r], t = et[r];
        if (f >= 0 && ein[r] == 0 && !(tg.mask(t, c0, per0) & (1 << f))) {
          int nb;
          if (f >= 2) {
            nb = tg.e0 + t + tg.face_off(f);
          } else {
            const int i = tg.i0 + t;
            nb = tg.e0 + t + ((f == 0) ? (i > 0 ? -1 : c0 - 1) : (i < c0 - 1 ? 1 : -(c0 - 1)));
          }
          const double* src = uo + (int64_t)nb * NV;
#pragma unroll
          for (int j = 0; j < NWC; ++j) gv[r][j] = __ldg(src + eoff[r][j]);
        }
      }
    };
    gather(0);
    int prev_e0 = 0, prev_nt = 0;
    for (int it = 0; it < n_my; ++it) {
      const int stage = it % NS;
      const int ob = it & 1;
      const double* sst = sm + stage * C::STAGE;
      const double* ust = sst + TILE;
      double* qb_w = q_s + ob * QE;
      mbar_wait(&full_bar[stage], (it / NS) & 1);
      const int fast = mfast_s[stage];
      // ---- q for this tile (TraceSnapshot of the neighbours' iterate k)
#pragma unroll
      for (int r = 0; r < QPT; ++r) {
        if (ef[r] >= 0) {
          const int t = et[r];
          double v = 0.0;
          if (!(mmask_s[stage][t] & (1 << ef[r]))) {
            if (ein[r] != 0) {
              const double* src = ust + (t + ein[r]) * NV;
#pragma unroll
              for (int j = 0; j < NWC; ++j) v = fma(ew[r][j], src[eoff[r][j]], v);
            } else {
#pragma unroll
              for (int j = 0; j < NWC; ++j) v = fma(ew[r][j], gv[r][j], v);
            }
          }
          qb_w[eq[r]] = v;
        }
      }
      // the out buffer ob was last stored for tile it-2: that store must have
      // read it before anyone writes the epilogue of tile it
      if (ctid == 0 && it >= 2) bulk_wait_read<0>();
      named_bar_sync(2, NCW * 32);   // q complete, out buffer free, epilogue of it-1 done
      if (ctid == 0 && it >= 1) {
        bulk_s2g(un + (int64_t)prev_e0 * NV, out_s + (ob ^ 1) * TILE, (uint32_t)(prev_nt * NV * sizeof(double)));
        bulk_commit();
      }
      gather(it + 1);   // lands during the contraction
      // ---- contraction u^{k+1} = s + L q
      double acc[NEG][RTW][2];
#pragma unroll
      for (int eg = 0; eg < NEG; ++eg) {
        const int te = ws_elem<NEG>(lane & 3, eg, 0);
#pragma unroll
        for (int j = 0; j < RTW; ++j) {
          const int row = (warp + j * NCW) * 8 + (lane >> 2);
          const bool ok = row < NV && (warp + j * NCW) < NRT;
          acc[eg][j][0] = ok ? sst[te * NV + row] : 0.0;
          acc[eg][j][1] = ok ? sst[(te + 1) * NV + row] : 0.0;
        }
      }
      const double* qb = qb_w + (lane >> 2) * KC + (lane & 3);
      if (fast) {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          double b[NEG];
#pragma unroll
          for (int eg = 0; eg < NEG; ++eg) b[eg] = qb[eg * 8 * KC + 4 * ks];
#pragma unroll
          for (int eg = 0; eg < NEG; ++eg)
#pragma unroll
            for (int j = 0; j < RTW; ++j) dmma_8x8x4(acc[eg][j][0], acc[eg][j][1], Lf[j][ks], b[eg]);
        }
      } else {
        const unsigned cset = mcset_s[stage];
        for (unsigned rem = cset; rem != 0u; rem &= rem - 1u) {
          const int c = __ffs(rem) - 1;
          for (int ks = 0; ks < KS; ++ks) {
            const int k = 4 * ks + (lane & 3);
            const int col = cf_s[k / NF] * NF + (k % NF);
            double av[RTW];
#pragma unroll
            for (int j = 0; j < RTW; ++j) {
              const int row = (warp + j * NCW) * 8 + (lane >> 2);
              av[j] = (row < NV) ? __ldg(a.LT + ((size_t)c * (NFACE * NF) + col) * NV + row) : 0.0;
            }
#pragma unroll
            for (int eg = 0; eg < NEG; ++eg) {
              const int n = lane >> 2;
              const double b = (mcls_s[stage][ws_elem<NEG>(n >> 1, eg, n & 1)] == c) ? qb[eg * 8 * KC + 4 * ks] : 0.0;
#pragma unroll
              for (int j = 0; j < RTW; ++j) dmma_8x8x4(acc[eg][j][0], acc[eg][j][1], av[j], b);
            }
          }
        }
      }
      // ---- epilogue: u^{k+1} -> out buffer, delta -> norm slot
      double* outb = out_s + ob * TILE;
      const int slot = it % NDB;
      double* dcur = d_s + slot * TILE;
      if (it >= NDB) mbar_wait(&dfree_bar[slot], ((it / NDB) - 1) & 1);
#pragma unroll
      for (int eg = 0; eg < NEG; ++eg) {
        const int te = ws_elem<NEG>(lane & 3, eg, 0);
#pragma unroll
        for (int j = 0; j < RTW; ++j) {
          const int row = (warp + j * NCW) * 8 + (lane >> 2);
          if (row < NV && (warp + j * NCW) < NRT) {
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int t = te + v;
              outb[t * NV + row] = acc[eg][j][v];
              dcur[t * NV + row] = acc[eg][j][v] - ust[t * NV + row];
            }
          }
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty_bar[stage]);
        mbar_arrive(&dfull_bar[slot]);
      }
      if (ctid == 0) {
        STile<D> tc;
        tc.init(a.g, (int)blockIdx.x + it * (int)gridDim.x, E, nlay, lsi);
        prev_e0 = tc.e0;
        prev_nt = tc.nt;
      }
    }
    // drain: store of the last tile
    named_bar_sync(2, NCW * 32);
    if (ctid == 0 && n_my >= 1) {
      bulk_s2g(un + (int64_t)prev_e0 * NV, out_s + ((n_my - 1) & 1) * TILE, (uint32_t)(prev_nt * NV * sizeof(double)));
      bulk_commit();
      bulk_wait<0>();
    }
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
