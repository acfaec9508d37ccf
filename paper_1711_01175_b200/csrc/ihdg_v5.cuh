// iHDG-II sweep, version 5: the register-tiled design of k_sweep_v4 for 2D
// problems with all four faces coupled and up to two weighted components per
// face scalar (BASELINE configs 2 and 3: convection-diffusion / shallow water,
// p=4, 75 DOFs per element).
//
// One warp owns one 8-element tile end to end, no helper warps, latency hidden
// by occupancy (16 warps per SM):
//   * s -> the DMMA accumulators (D fragment: row = lane>>2, two elements per
//     lane), straight from global memory;
//   * q -> the B fragment.  The k index is dealt as k slot (step ks, lane&3) =
//     (face node ks, coupled face lane&3), so a lane gathers the N1 nodes of
//     ONE face of ONE element (element lane>>2): one neighbour index per lane
//     and tile, NWC weighted components per node, all issued before the first
//     use and branch-free (a missing neighbour reads the element itself with
//     weight 0).  The columns of L are permuted alike;
//   * u^k -> a warp-private staging tile by one TMA bulk copy (the tile is
//     contiguous), read back in the epilogue for delta = u^{k+1} - u^k;
//   * L (interior class) in shared memory in A-fragment order; mixed-class
//     tiles (domain boundary) take one masked pass per class with L from L2;
//   * u^{k+1} stored from registers; delta -> a warp-private scratch tile and
//     the exact triangular DFMA passes of the mass-weighted norm (k_sweep_v3's).
//
// PF consecutive warps (a group) own the PF physical tiles of one logical tile
// (the generic kernel's tile: one tile partial), combined in warp order through
// a named barrier one iteration late.  Launched with programmatic stream
// serialization (see pdl_wait).
//
// HBM per element-DOF: s, u^k, u^{k+1} = 24 B.
#pragma once

#include <climits>

#include "ihdg_stream.cuh"

namespace ihdg {

template <int N1, int M, int NWC, int NW, int PF>
struct V5Cfg {
  static constexpr int D = 2, NCF = 4;
  static constexpr int E = 8;                     // elements per physical tile (DMMA n)
  static constexpr int NP = N1 * N1;
  static constexpr int NV = M * NP;
  static constexpr int NF = N1;
  static constexpr int NFACE = 4;
  static constexpr int NRT = (NV + 7) / 8;        // DMMA row tiles
  static constexpr int KS = NF;                   // DMMA k steps: one face node per step, four faces per step
  static constexpr int NT = 32 * NW;
  static constexpr int NG = NW / PF;              // groups (logical tiles in flight) per CTA
  static constexpr int TILE = E * NV;             // doubles, contiguous in global memory
  static constexpr int TILEP = (TILE + 1) / 2 * 2;
  static constexpr int LFR = NRT * KS * 32;       // L fragments (doubles)
  static constexpr int N_DBL = LFR + NW * 2 * TILEP;   // + per warp: u^k staging tile, delta scratch tile
  static constexpr size_t BYTES = (size_t)N_DBL * sizeof(double);
  static constexpr int LPL = NP / N1;             // norm lines per (element, component) and axis
  static constexpr int NLINES = E * M * LPL;
  static_assert((TILE * sizeof(double)) % 16 == 0, "tile bytes must be 16-byte multiples (bulk copy)");
  static_assert(NW % PF == 0 && NG >= 1 && NG <= 15, "one named barrier per group");
  static_assert(BYTES + 4096 + 1024 <= 233472, "shared memory over the sm_100a limit");
};

template <int N1, int M, int NWC, int NW, int PF>
__global__ void __launch_bounds__(V5Cfg<N1, M, NWC, NW, PF>::NT, 1) k_sweep_v5(const ihdg_sweep_args a) {
  using C = V5Cfg<N1, M, NWC, NW, PF>;
  constexpr int D = 2, E = C::E, NP = C::NP, NV = C::NV, NF = C::NF, NFACE = C::NFACE;
  constexpr int NRT = C::NRT, KS = C::KS;

  extern __shared__ __align__(16) double sm[];
  const double* lfr_s = sm;

  __shared__ double chol_s[N1 * N1];
  __shared__ double cw_s[IHDG_MAX_COMP];
  __shared__ int com_s[64];                 // class_of_mask
  __shared__ double part_s[C::NG][2][PF];
  __shared__ int last_s;
  __shared__ __align__(8) uint64_t ubar[NW];   // per warp: u^k tile landed

  ihdg_iter_state* st = a.state;
  pdl_launch_dependents();   // the next launch may start its own prologue

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (lane == 0) {
    mbar_init(&ubar[warp], 1);
    fence_mbar_init();   // visible to the async proxy after the setup barrier below
  }
  Geo geo;
  geo.init(a.g, E * PF);  // logical tile = PF physical tiles = the generic kernel's tile
  const int64_t ls = geo.ls;
  const double* __restrict__ uo = a.u_old + ls * NV;
  double* __restrict__ un = a.u_new + ls * NV;
  const int fast_class = a.class_of_mask[0];

  for (int i = tid; i < N1 * N1; i += blockDim.x) chol_s[i] = a.chol1d[i];
  if (tid < IHDG_MAX_COMP) cw_s[tid] = a.comp_w[tid];
  if (tid < 64) com_s[tid] = a.class_of_mask[tid];
  // interior-class L in DMMA A-fragment order with the k permutation: frag
  // (rt, ks), lane l -> L[8 rt + (l>>2)][column of (face l&3, node ks)]
  for (int idx = tid; idx < C::LFR; idx += blockDim.x) {
    const int l = idx & 31, fr = idx >> 5;
    const int rt = fr / KS, ks = fr - (fr / KS) * KS;
    const int row = rt * 8 + (l >> 2);
    const int col = (l & 3) * NF + ks;
    sm[idx] = (row < NV) ? a.LT[((size_t)fast_class * (NFACE * NF) + col) * NV + row] : 0.0;
  }
  __syncthreads();
  // everything above reads only launch-invariant data (operators, tables);
  // the iterate, s and the iteration state belong to the previous launches
  pdl_wait();
  if (st->status != IHDG_RUNNING) return;

  const int grp = warp / PF, sub = warp - grp * PF;
  const int nlog = (int)geo.ntiles;
  const int nlay = (int)(a.g.layer_end - a.g.layer_begin);
  const int lsi = (int)ls;
  const int c0 = (int)a.g.cells[0];
  const int per0 = a.g.periodic[0];
  const int kk = lane & 3;            // B fragment: this lane's face; D fragment: element pair
  const int te = 2 * kk;              // D-fragment columns (elements) of this lane
  const int rsub = lane >> 2;         // D-fragment row inside a row tile; B-fragment element
  double* uks = sm + C::LFR + warp * 2 * C::TILEP;   // u^k staging tile (TMA only)
  double* scr = uks + C::TILEP;                      // delta scratch tile
  FastDiv dsegs0, dc1;
  dsegs0.init((uint32_t)(c0 / E));
  dc1.init(1u);
  const int segs0 = c0 / E;

  // this lane's face f = kk: weighted components and source node offsets inside
  // the neighbour (its face f^1), node ks in k step ks
  int wcomp[NWC];
  double wval[NWC];
  {
    int j = 0;
    for (int c = 0; c < M && j < NWC; ++c)
      if (a.face_w[kk][c] != 0.0) {
        wcomp[j] = c;
        wval[j] = a.face_w[kk][c];
        ++j;
      }
    for (; j < NWC; ++j) {
      wcomp[j] = 0;
      wval[j] = 0.0;
    }
  }
  // source node of step ks on face f^1: x faces (f < 2): (i = 0 or N1-1, j = ks);
  // y faces: (i = ks, j = 0 or N1-1)
  const int nbase = kk < 2 ? ((kk ^ 1) & 1) * (N1 - 1) : ((kk ^ 1) & 1) * (N1 - 1) * N1;
  const int nstep = kk < 2 ? N1 : 1;

  auto group_partial = [&](int lt_done, int it_done) {
    if constexpr (PF == 1) {
      if (lane == 0) a.tile_partials[lt_done] = a.jac * part_s[grp][it_done & 1][0];
    } else {
      named_bar_sync(1 + grp, 32 * PF);
      if (sub == 0 && lane == 0) {
        double p = 0.0;
#pragma unroll
        for (int w = 0; w < PF; ++w) p += part_s[grp][it_done & 1][w];
        a.tile_partials[lt_done] = a.jac * p;
      }
    }
  };
  int itn = 0, prev_lt = -1;
  for (int lt = (int)blockIdx.x * C::NG + grp; lt < nlog; lt += (int)gridDim.x * C::NG, ++itn) {
    STile<D> ti;
    ti.init(a.g, lt * PF + sub, E, nlay, lsi, segs0, dsegs0, dc1);
    const int e0 = ti.e0;
    // ---- operand loads, all independent ----
    double acc[NRT][2], b[KS];
    {
      const double* sg = a.s + (int64_t)(e0 + te) * NV + rsub;
#pragma unroll
      for (int rt = 0; rt < NRT; ++rt) {
        const bool ok = rt * 8 + rsub < NV;
        acc[rt][0] = ok ? __ldcs(sg + rt * 8) : 0.0;
        acc[rt][1] = ok ? __ldcs(sg + NV + rt * 8) : 0.0;
      }
    }
    // u^k tile -> the staging tile by the TMA unit (the tile is contiguous).
    // The region is never written through the generic proxy, so no proxy
    // fence is needed; __syncwarp orders the read-back of the previous tile.
    __syncwarp();
    if (lane == 0) {
      mbar_arrive_expect_tx(&ubar[warp], (uint32_t)(C::TILE * sizeof(double)));
      bulk_g2s(uks, uo + (int64_t)e0 * NV, (uint32_t)(C::TILE * sizeof(double)), &ubar[warp]);
    }
    {
      // neighbour of element rsub across this lane's face kk
      constexpr int NONE = INT_MIN;   // ghost-layer neighbours have negative local indices
      const int i = ti.i0 + rsub;
      int nb;
      if (kk == 0) nb = (!per0 && i == 0) ? NONE : e0 + rsub + (i > 0 ? -1 : c0 - 1);
      else if (kk == 1) nb = (!per0 && i == c0 - 1) ? NONE : e0 + rsub + (i < c0 - 1 ? 1 : -(c0 - 1));
      else if (kk == 2) nb = ti.has[2] ? e0 + rsub + ti.off[2] : NONE;
      else nb = ti.has[3] ? e0 + rsub + ti.off[3] : NONE;
      const double wz = nb != NONE ? 1.0 : 0.0;
      const double* src = uo + (int64_t)(nb != NONE ? nb : e0 + rsub) * NV + nbase;
      double g[KS][NWC];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int j = 0; j < NWC; ++j) g[ks][j] = __ldg(src + wcomp[j] * NP + ks * nstep);
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < NWC; ++j) v = fma(wval[j], g[ks][j], v);
        b[ks] = v * wz;
      }
    }
    if (prev_lt >= 0) group_partial(prev_lt, itn - 1);
    // ---- operator classes of the tile ----
    const int mycls = com_s[ti.mask(rsub, c0, per0)];
    const int fast = __all_sync(0xffffffffu, mycls == fast_class);
    if (fast) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int rt = 0; rt < NRT; ++rt) dmma_8x8x4(acc[rt][0], acc[rt][1], lfr_s[(rt * KS + ks) * 32 + lane], b[ks]);
      }
    } else {
      // one masked pass per operator class present in the tile
      unsigned cset = (mycls >= 0 && mycls < 32) ? (1u << mycls) : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cset |= __shfl_xor_sync(0xffffffffu, cset, o);
      for (unsigned rem = cset; rem != 0u; rem &= rem - 1u) {
        const int c = __ffs(rem) - 1;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const double bb = (mycls == c) ? b[ks] : 0.0;
          const double* Lc = a.LT + ((size_t)c * (NFACE * NF) + kk * NF + ks) * NV;
#pragma unroll
          for (int rt = 0; rt < NRT; ++rt) {
            const int row = rt * 8 + rsub;
            dmma_8x8x4(acc[rt][0], acc[rt][1], (row < NV) ? __ldg(Lc + row) : 0.0, bb);
          }
        }
      }
    }
    // ---- u^{k+1} -> global (64-byte runs), delta -> scratch ----
    {
      double* ug = un + (int64_t)(e0 + te) * NV + rsub;
#pragma unroll
      for (int rt = 0; rt < NRT; ++rt)
        if (rt * 8 + rsub < NV) {
          __stcs(ug + rt * 8, acc[rt][0]);
          __stcs(ug + NV + rt * 8, acc[rt][1]);
        }
    }
    mbar_wait(&ubar[warp], itn & 1);   // the u^k tile has landed
#pragma unroll
    for (int rt = 0; rt < NRT; ++rt) {
      const int row = rt * 8 + rsub;
      if (row < NV) {
        scr[te * NV + row] = acc[rt][0] - uks[te * NV + row];
        scr[(te + 1) * NV + row] = acc[rt][1] - uks[(te + 1) * NV + row];
      }
    }
    __syncwarp();
    // ||delta||_M^2 = J |(C^T x C^T) delta|^2, M1 = C C^T: one exact triangular
    // pass per axis over the lines of the node grid (in place)
    double nsum = 0.0;
    int mul = 1;
#pragma unroll
    for (int ax = 0; ax < D; ++ax) {
      const bool last_ax = ax == D - 1;
#pragma unroll
      for (int m = 0; m < (C::NLINES + 31) / 32; ++m) {
        const int ln = lane + 32 * m;
        if (ln < C::NLINES) {
          const int t = ln / (M * C::LPL);
          const int c = (ln / C::LPL) % M;
          const int rem = ln % C::LPL;
          const int base = t * NV + c * NP + rem * (ax == 0 ? N1 : 1);
          double x[N1];
#pragma unroll
          for (int i = 0; i < N1; ++i) x[i] = scr[base + i * mul];
          double sq = 0.0;
#pragma unroll
          for (int i = 0; i < N1; ++i) {
            double y = 0.0;
#pragma unroll
            for (int ip = i; ip < N1; ++ip) y = fma(chol_s[ip * N1 + i], x[ip], y);
            if (last_ax) sq = fma(y, y, sq);
            else scr[base + i * mul] = y;
          }
          if (last_ax) nsum = fma(cw_s[c], sq, nsum);
        }
      }
      __syncwarp();
      mul *= N1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, o);
    if (lane == 0) part_s[grp][itn & 1][sub] = nsum;
    prev_lt = lt;
  }
  if (prev_lt >= 0) group_partial(prev_lt, itn - 1);

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
