// Warp-specialised iHDG-II sweep for 2D configurations (production path for
// BASELINE configs 2, 3 and 5).  The roles run asynchronously and hand tiles
// over through mbarriers only (no CTA-wide barrier in the steady state):
//
//   producer warp  : per tile, metadata + TMA bulk copies of the s and u^k
//                    tiles + cp.async gathers of out-of-tile neighbour faces
//                    into an NS-stage ring                   -> full[stage]
//   prep warps (4) : neighbour face scalars q (TraceSnapshot) for the stage
//                    -> qready[stage]; then, one tile behind, the bulk store
//                    of u^{k+1} and the fixed-order tile partial of the norm
//   consumer warps : DMMA contraction u^{k+1} = s + L q (L fragments in
//                    registers) for tile i interleaved with the tensor-core
//                    norm J |C^T Delta C|^2 of tile i-1      -> done[i&1]
#pragma once

#include "ihdg_stream.cuh"

namespace ihdg {

#ifndef IHDG_WS_LAG
#define IHDG_WS_LAG 1   // the norm of tile i-LAG runs in iteration i (2 measured no gain)
#endif
#ifndef IHDG_WS_PF
#define IHDG_WS_PF 0   // L2 prefetch distance in tiles (0 = off; 1/2/4 measured no gain)
#endif
#ifdef IHDG_MEMONLY
#define IHDG_MEMONLY_ON 1   // data-movement-only build (A/B experiment)
#else
#define IHDG_MEMONLY_ON 0
#endif

// Element <-> DMMA column map of the consumers: column 2a+v of element group
// eg (a = lane & 3 for the accumulators) holds element a*2*NEG + 2*eg + v.
// With an odd element stride NV the four elements a half-warp touches then
// sit 4*NV = 4 (mod 16) double-banks apart: s, u^k and u^{k+1} tile accesses
// are conflict-free without padding the TMA-copied tiles.
template <int NEG>
__device__ __forceinline__ int ws_elem(int a, int eg, int v) { return a * 2 * NEG + 2 * eg + v; }
// column slot (eg * 8 + n) of element t: q is stored in column order so the
// B-operand loads stay conflict-free
template <int NEG>
__device__ __forceinline__ int ws_qcol(int t) {
  const int a = t / (2 * NEG), r = t - a * 2 * NEG;
  return (r >> 1) * 8 + 2 * a + (r & 1);
}
// swizzled offset of node (kk, nn) inside a delta unit
__device__ __forceinline__ int ws_dnode(int kk, int nn) { return kk * 8 + (nn ^ (4 * ((kk >> 1) & 1))); }

// Norm units (element, component) of consumer warp w: units [first, first +
// cnt).  The warps of one SM sub-partition (warp % 4) share one fp64 tensor
// pipe (16 clk per DMMA, tools/microbench/dmma_smsp.cu), 10 consumer warps sit
// 3/3/2/2 on them, and the consumers run the norm of a tile in lockstep (it
// needs every warp's delta): the phase lasts as long as the busiest
// sub-partition, so the units are dealt evenly per sub-partition (12 each for
// 48 units), not per warp.
template <int NCW, int NRT, int KS, int NEG, int NU>
__host__ __device__ constexpr void ws_units(int w, int& first, int& cnt) {
  int load[4] = {0, 0, 0, 0};
  int uc[NCW] = {};
  for (int u = 0; u < NU; ++u) {
    int best = 0;
    for (int i = 1; i < NCW; ++i)
      if (load[i % 4] < load[best % 4] || (load[i % 4] == load[best % 4] && uc[i] < uc[best])) best = i;
    ++uc[best];
    ++load[best % 4];
  }
  first = 0;
  for (int i = 0; i < w; ++i) first += uc[i];
  cnt = uc[w];
}
// the deal as a compile-time table (the greedy loop costs ~10 us per launch
// when every consumer thread runs it)
template <int NCW>
struct WsUnitTable {
  int first[NCW], cnt[NCW];
};
template <int NCW, int NRT, int KS, int NEG, int NU>
__host__ __device__ constexpr WsUnitTable<NCW> ws_unit_table() {
  WsUnitTable<NCW> t{};
  for (int w = 0; w < NCW; ++w) ws_units<NCW, NRT, KS, NEG, NU>(w, t.first[w], t.cnt[w]);
  return t;
}
template <int NCW, int NRT, int KS, int NEG, int NU>
__host__ __device__ constexpr int ws_max_units() {
  int mx = 0;
  for (int w = 0; w < NCW; ++w) {
    int f = 0, c = 0;
    ws_units<NCW, NRT, KS, NEG, NU>(w, f, c);
    mx = c > mx ? c : mx;
  }
  return mx;
}

// tensor-core norm over the swizzled delta tile: units u0 .. u0 + ucnt - 1 of
// this warp, (element, component); sum of w_c |C^T Delta C|_F^2
// The second product Y = R C contracts over the columns of R in the order the
// D fragment holds them (k slot (ks, c) = column 2 c + ks, with C's rows
// permuted alike in cfp), so R feeds the A operand straight from the
// accumulator registers: no shuffles between the two DMMAs.
template <int N1, int M, int E, int UPW, int DUE, int DUC>
__device__ __forceinline__ double norm_units_swz(const double* __restrict__ dbuf, int u0, int ucnt, int lane,
                                                 const double (&cfr)[2], const double (&cfp)[2],
                                                 const double* comp_w) {
  double acc = 0.0;
  double r0[UPW], r1[UPW];
#pragma unroll
  for (int m = 0; m < UPW; ++m) {
    r0[m] = 0.0;
    r1[m] = 0.0;
    if (m < ucnt) {   // warp-uniform
      const int u = u0 + m;
      const int t = u / M, c = u - (u / M) * M;
      const double* base = dbuf + t * DUE + c * DUC;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int kk = 4 * ks + (lane & 3), nn = lane >> 2;
        const double b = (kk < N1 && nn < N1) ? base[ws_dnode(kk, nn)] : 0.0;
        dmma_8x8x4(r0[m], r1[m], cfr[ks], b);   // R = C^T Delta
      }
    }
  }
#pragma unroll
  for (int m = 0; m < UPW; ++m) {
    if (m < ucnt) {
      const int c = (u0 + m) % M;
      double y0 = 0.0, y1 = 0.0;
      dmma_8x8x4(y0, y1, r0[m], cfp[0]);  // Y = R C, columns 2c of R
      dmma_8x8x4(y0, y1, r1[m], cfp[1]);  // columns 2c + 1
      const double w = comp_w[c];
      acc = fma(w * y0, y0, acc);
      acc = fma(w * y1, y1, acc);
    }
  }
  return acc;
}

template <int N1, int M, int NCF, int NWC, int E, int NS, bool GRAM = false>
struct WCfg {
  static constexpr int D = 2;
  static constexpr int NP = N1 * N1;
  static constexpr int NV = M * NP;
  static constexpr int NF = N1;
  static constexpr int KC = NCF * NF;
  static constexpr int NRT = (NV + 7) / 8;
  static constexpr int KS = KC / 4;
  static constexpr int NEG = E / 8;
#ifdef IHDG_WS_NCW
  static constexpr int NCW = IHDG_WS_NCW;                          // A/B builds
#else
  static constexpr int NCW = NRT >= 16 ? 10 : (NRT >= 8 ? 8 : 4);  // consumer warps
#endif
  static constexpr int RTW = (NRT + NCW - 1) / NCW;
  static constexpr int UPW = ws_max_units<NCW, NRT, KS, NEG, E * M>();   // most norm units of one warp
#ifdef IHDG_WS_NQW
  static constexpr int NQW = IHDG_WS_NQW;                          // A/B builds
#else
  static constexpr int NQW = 4;                                    // prep warps
#endif
  static constexpr int NT = 32 * (NCW + NQW + 1);
  static constexpr int TILE = E * NV;
  static constexpr int HALO = 0;   // out-of-tile faces: prep warps load them into registers
  static constexpr int QT = E * KC;
  // stage: s tile, u^k tile, q (neighbour face scalars), dq = q^k - q^{k-1}
  // (Gram-form norm), the last two in the consumers' column order
  static constexpr int STAGE = 2 * TILE + HALO + (GRAM ? 2 : 1) * QT;
  // Gram-form norm ||R dq||^2: R is KC x KC upper triangular, so row tile rt
  // of R touches k-steps 2 rt .. KS-1; one (row tile, element group) item per
  // consumer warp, the heavy items on the last warps (lightest contraction)
  static constexpr int GRT = (KC + 7) / 8;
  static constexpr int NGI = GRT * NEG;
  static constexpr int OFF_OUT = NS * STAGE;
  // delta tiles: bank-conflict-free swizzled layout (node row stride 8,
  // column XOR 4 on every other pair of rows; component stride DUC, element
  // stride DUE), written by the epilogue and read by the norm
  static constexpr int DUC = 8 * N1 + 3;
  static constexpr int DUE = M * DUC;
  static constexpr int DT = E * DUE;
  // delta/partial rings: in iteration i a warp knows every warp has finished
  // iteration i-LAG, i.e. the norms up to tile i-2 LAG, so 2 LAG slots keep
  // every slot's readers done before it is rewritten
  static constexpr int LAG = IHDG_WS_LAG;
  static constexpr int NDB = 2 * LAG;
  static constexpr int OFF_D = OFF_OUT + 2 * TILE;
  static constexpr int OFF_RED = OFF_D + NDB * DT;
  // per-warp norm partials: slot = tile % NRED.  A Gram partial of tile j is
  // written in iteration j, a direct one in j + 1, and prep warp 0 reads it in
  // its iteration j + 2; consumers reach iteration j + NRED only after prep
  // iteration j + NRED started, so NRED = 4 slots never overwrite an unread one
  static constexpr int NRED = 4;
  static constexpr int N_DBL = OFF_RED + 32 * NRED;
  static constexpr int NBAR = 3 * NS + 4;
  static constexpr size_t BYTES = (size_t)N_DBL * sizeof(double) + NBAR * sizeof(uint64_t);
  static_assert(KC % 4 == 0 && E % 8 == 0 && E <= 32 && N1 <= 8, "ws config");
  static_assert((TILE * sizeof(double)) % 16 == 0, "tile bytes must be 16-byte multiples");
  static_assert(E % NQW == 0, "prep warps split the tile");
  static_assert(NGI <= NCW, "one Gram item per consumer warp");
  static_assert(BYTES + 4096 <= 232448, "shared memory (dynamic + static) over the sm_100a opt-in limit");
};

// GRAM: the instantiation that stores q and takes the Gram-form norm from the
// second sweep of a solve on (ihdg.h, q_store); without it the code is the
// direct-norm kernel only (no q stores, no dq slots in the stages).
template <int N1, int M, int NCF, int NWC, int E, int NS, bool GRAM>
__global__ void __launch_bounds__(WCfg<N1, M, NCF, NWC, E, NS, GRAM>::NT, 1)
    k_sweep_ws(const ihdg_sweep_args a) {
  using C = WCfg<N1, M, NCF, NWC, E, NS, GRAM>;
  constexpr int D = 2, NP = C::NP, NV = C::NV, NF = C::NF, NFACE = 4, KC = C::KC;
  constexpr int NRT = C::NRT, KS = C::KS, NEG = C::NEG, NCW = C::NCW, RTW = C::RTW, UPW = C::UPW;
  constexpr int NQW = C::NQW, TILE = C::TILE;

  extern __shared__ __align__(16) double sm[];
  double* out_s = sm + C::OFF_OUT;
  double* d_s = sm + C::OFF_D;
  double* red_s = sm + C::OFF_RED;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::N_DBL);
  uint64_t* full_bar = bars;             // [NS] producer -> prep
  uint64_t* qready_bar = bars + NS;      // [NS] prep -> consumers
  uint64_t* empty_bar = bars + 2 * NS;   // [NS] consumers -> producer
  uint64_t* done_bar = bars + 3 * NS;    // [2]  consumers -> prep, consumers
  uint64_t* outfree_bar = done_bar + 2;  // [2]  prep -> consumers

  __shared__ int fv_s[NFACE][NF];
  __shared__ int cf_s[NCF];
  __shared__ int wc_s[NCF][NWC];
  __shared__ double ww_s[NCF][NWC];
  __shared__ double chol_s[N1 * N1];
  __shared__ int qf_s[KC], qh_s[KC];
  __shared__ int qt_s[KC][NWC];
  __shared__ long long me0_s[NS];
  __shared__ int mnt_s[NS], mfast_s[NS];
  __shared__ unsigned mcset_s[NS];
  __shared__ int mmask_s[NS][E], mcls_s[NS][E];
  __shared__ int tile_s[NS];
  __shared__ int com_s[64];
  __shared__ int last_s;

  ihdg_iter_state* st = a.state;
  if (st->status != IHDG_RUNNING) return;
  V3_DECL

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  Geo geo;
  geo.init(a.g, E);
  const int64_t ls = geo.ls;
  const double* __restrict__ uo = a.u_old + ls * NV;
  double* __restrict__ un = a.u_new + ls * NV;

  for (int i = tid; i < NFACE * NF; i += blockDim.x) fv_s[i / NF][i % NF] = face_node_vidx(D, N1, i / NF, i % NF);
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
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&qready_bar[s], NQW);
      mbar_init(&empty_bar[s], NCW);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&done_bar[b], NCW);
      mbar_init(&outfree_bar[b], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (tid < KC) {   // one thread per neighbour scalar (was a serial loop of thread 0)
    const int k = tid;
    const int ci = k / NF, nn = k % NF, f = cf_s[ci];
    qf_s[k] = f;
    for (int j = 0; j < NWC; ++j) qt_s[k][j] = wc_s[ci][j] * NP + face_node_vidx(D, N1, f ^ 1, nn);
    qh_s[k] = ci * NWC * NF + nn;
  }
  __syncthreads();

  const int fast_class = a.class_of_mask[0];
  const int ntiles = (int)geo.ntiles;
  // Gram-form norm (ihdg.h, q_store): q of every tile is stored each sweep;
  // the stored q^{k-1} is used from the second sweep of a solve on (the
  // last CTA's finalize of the previous launch wrote iters; no CTA of this
  // launch can finalize before every CTA has read it)
  constexpr bool qsave = GRAM;   // dispatch guarantees q_store / gram_kc
  const bool gram = GRAM && a.gram_R != nullptr && st->iters > 0;
  V3_T0(tk0);
  int n_my = 0;  // tiles of this CTA
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) ++n_my;

  if (warp == NCW + NQW) {
    // ============================ producer warp ============================
    const int c0 = (int)a.g.cells[0];
    const int per0 = a.g.periodic[0];
    const int nlay = (int)(a.g.layer_end - a.g.layer_begin);
    const int lsi = (int)ls;
    for (int it = 0; it < n_my; ++it) {
      const int tile = blockIdx.x + it * gridDim.x;
      const int stage = it % NS;
      V3_T0(tw);
      WS_STAMP(warp, it, 0);
      if (it >= NS) mbar_wait(&empty_bar[stage], ((it / NS) - 1) & 1);
      WS_STAMP(warp, it, 1);
      V3_ACC(0, tw);
      V3_T0(tl);
      double* sst = sm + stage * C::STAGE;
      double* ust = sst + TILE;
      STile<D> ti;
      ti.init(a.g, tile, E, nlay, lsi);
      const int e0 = ti.e0;
      const int nt = ti.nt;
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
        me0_s[stage] = e0;
        mnt_s[stage] = nt;
        mfast_s[stage] = fast;
        mcset_s[stage] = cset;
        tile_s[stage] = tile;
      }
      __syncwarp();
      if (lane == 0) {
        const uint32_t bytes = (uint32_t)(nt * NV * sizeof(double));
        constexpr uint32_t qbytes = (uint32_t)(C::QT * sizeof(double));
        mbar_arrive_expect_tx(&full_bar[stage], 2 * bytes + (gram ? qbytes : 0u));  // release: metadata above
        bulk_g2s(sst, a.s + (int64_t)e0 * NV, bytes, &full_bar[stage]);
        bulk_g2s(ust, uo + (int64_t)e0 * NV, bytes, &full_bar[stage]);
        // the stored q^{k-1} of the tile (consumer column order) into the dq slot
        if constexpr (GRAM)
          if (gram) bulk_g2s(ust + TILE + C::HALO + C::QT, a.q_store + (int64_t)tile * C::QT, qbytes, &full_bar[stage]);
      }
      if (IHDG_WS_PF > 0 && lane == 0 && it + IHDG_WS_PF < n_my) {
        // tile it+PF will be copied into a stage PF tiles from now: pull it into L2
        STile<D> tp;
        tp.init(a.g, tile + IHDG_WS_PF * (int)gridDim.x, E, nlay, lsi);
        const uint32_t pb = (uint32_t)(tp.nt * NV * sizeof(double));
        bulk_prefetch_l2(a.s + (int64_t)tp.e0 * NV, pb);
        bulk_prefetch_l2(uo + (int64_t)tp.e0 * NV, pb);
      }
      V3_ACC(9, tl);
      WS_STAMP(warp, it, 2);
    }
  } else if (warp >= NCW) {
    // ============================ prep warps ===============================
    const int pw = warp - NCW;
    const int c0 = (int)a.g.cells[0];
    const int per0 = a.g.periodic[0];
    const int nlay = (int)(a.g.layer_end - a.g.layer_begin);
    const int lsi = (int)ls;
    int prev_e0 = 0, prev_nt = 0;
    int hist[4] = {-1, -1, -1, -1};   // tile ids of the last iterations (it & 3)
    static_assert(C::LAG + 1 <= 4, "tile history");
    constexpr int HALF = E / NQW;
    constexpr int QM = (HALF * KC + 31) / 32;
    // out-of-tile neighbour face nodes of this warp's entries, loaded from
    // global (L2) into registers one tile ahead
    double gv[QM][NWC], gvn[QM][NWC];
    int qs = 0, ql = 0, qsn = 0, qln = 0;
    // per-lane entry constants, hoisted out of the tile loop: entry m of this
    // lane is (element t, column k) with k's face f and its gather offsets
    int ent_t[QM], ent_f[QM], ent_q[QM][NWC];
#pragma unroll
    for (int m = 0; m < QM; ++m) {
      const int idx = lane + 32 * m;
      const bool ok = idx < HALF * KC;
      const int k = ok ? idx - (idx / KC) * KC : 0;
      ent_t[m] = ok ? pw * HALF + idx / KC : -1;
      ent_f[m] = qf_s[k];
#pragma unroll
      for (int j = 0; j < NWC; ++j) ent_q[m][j] = qt_s[k][j];
    }
    auto gather = [&](int itg, double (&dst)[QM][NWC], int& in_bits, int& ld_bits) {
      in_bits = 0;
      ld_bits = 0;
      if (itg >= n_my) return;
      STile<D> tg;
      tg.init(a.g, (int)blockIdx.x + itg * (int)gridDim.x, E, nlay, lsi);
      // missing neighbours: faces of axes >= 1 are tile-uniform, x faces only
      // at the tile ends
      int hm = 0;
#pragma unroll
      for (int f = 2; f < 2 * D; ++f)
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
              in_bits |= 1 << m;
            } else {
              ld_bits |= 1 << m;
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
    gather(0, gv, qs, ql);
    for (int it = 0; it < n_my; ++it) {
      const int stage = it % NS;
      gather(it + 1, gvn, qsn, qln);
      V3_T0(tp);
      WS_STAMP(warp, it, 0);
      mbar_wait(&full_bar[stage], (it / NS) & 1);
      WS_STAMP(warp, it, 1);
      V3_ACC(1, tp);
      V3_T0(tq);
      // stage metadata is read now: the stage can be refilled once the
      // consumers release it, possibly before this warp stores the tile
      const int nt = mnt_s[stage];
      const int cur_e0 = (int)me0_s[stage];
      const int cur_tile = tile_s[stage];
      const double* sst = sm + stage * C::STAGE;
      const double* ust = sst + TILE;
      double* qst = const_cast<double*>(ust) + TILE + C::HALO;
      double* dqst = qst + C::QT;   // holds q^{k-1} (TMA), becomes dq in place
      double* qdst = qsave ? a.q_store + (int64_t)cur_tile * C::QT : nullptr;
#pragma unroll
      for (int m = 0; m < QM; ++m) {
        const int t = ent_t[m];
        if (t >= 0) {
          const int k = lane + 32 * m - (t - pw * HALF) * KC;
          const double* w = ww_s[k / NF];
          double v = 0.0;
          if (qs & (1 << m)) {
            const double* src = ust + (t + (ent_f[m] == 0 ? -1 : 1)) * NV;
#pragma unroll
            for (int j = 0; j < NWC; ++j) v = fma(w[j], src[ent_q[m][j]], v);
          } else if (ql & (1 << m)) {
#pragma unroll
            for (int j = 0; j < NWC; ++j) v = fma(w[j], gv[m][j], v);
          }
          const int qi = ws_qcol<C::NEG>(t) * KC + k;
          qst[qi] = v;
          if constexpr (GRAM) {
            if (gram) dqst[qi] = v - dqst[qi];
            __stcs(qdst + qi, v);   // q store: the stage's column order
          }
        }
      }
      if constexpr (GRAM)
        if (gram) fence_proxy_async();   // dq overwrote a TMA destination; the stage is refilled by TMA
      __syncwarp();
      V3_ACC(2, tq);
      WS_STAMP(warp, it, 2);
      if (lane == 0) mbar_arrive(&qready_bar[stage]);
      if (it >= 1) {
        const int pb = (it - 1) & 1;
        mbar_wait(&done_bar[pb], ((it - 1) >> 1) & 1);
        WS_STAMP(warp, it, 3);
        if (pw == 0 && lane == 0) {
          bulk_s2g(un + (int64_t)prev_e0 * NV, out_s + pb * TILE, (uint32_t)(prev_nt * NV * sizeof(double)));
          bulk_commit();
          if (it >= 2) {
            bulk_wait_read<1>();                       // store of tile it-2 has read its buffer
            mbar_arrive(&outfree_bar[it & 1]);
          }
        }
        if (pw == 0 && lane == 1) {
          const int jt = it - 1 - C::LAG;   // every warp has reduced tile jt by done(it-1)
          if (jt >= 0) {
            double s = 0.0;
            for (int w = 0; w < NCW; ++w) s += red_s[(jt % C::NRED) * 32 + w];
            a.tile_partials[hist[jt & 3]] = a.jac * s;
          }
        }
      }
      hist[it & 3] = cur_tile;
      prev_e0 = cur_e0;
      prev_nt = nt;
      // the gathers of tile it+1 are consumed only here (a register move
      // waits on the load), i.e. after qready(it) and the done wait
#pragma unroll
      for (int m = 0; m < QM; ++m)
#pragma unroll
        for (int j = 0; j < NWC; ++j) gv[m][j] = gvn[m][j];
      qs = qsn;
      ql = qln;
    }
    // drain: store of the last tile, partial of the one before
    if (n_my >= 1) {
      const int L = n_my - 1;
      mbar_wait(&done_bar[L & 1], (L >> 1) & 1);
      if (pw == 0 && lane == 0) {
        bulk_s2g(un + (int64_t)prev_e0 * NV, out_s + (L & 1) * TILE, (uint32_t)(prev_nt * NV * sizeof(double)));
        bulk_commit();
        const int jt = L - C::LAG;
        if (jt >= 0) {
          double s = 0.0;
          for (int w = 0; w < NCW; ++w) s += red_s[(jt % C::NRED) * 32 + w];
          a.tile_partials[hist[jt & 3]] = a.jac * s;
        }
        bulk_wait<0>();
      }
    }
  } else {
    // ============================ consumer warps ===========================
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
    int doff[RTW];   // swizzled delta offset of this lane's row in each row tile
#pragma unroll
    for (int j = 0; j < RTW; ++j) {
      const int row = (warp + j * NCW) * 8 + (lane >> 2);
      const int r = row < NV ? row : 0;
      const int c = r / NP, node = r - c * NP;
      doff[j] = c * C::DUC + ws_dnode(node / N1, node - (node / N1) * N1);
    }
    double cfr[2];
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int kk = 4 * ks + (lane & 3), nn = lane >> 2;
      cfr[ks] = (kk < N1 && nn < N1) ? chol_s[kk * N1 + nn] : 0.0;
    }
    double cfp[2];   // C rows in the D-fragment column order: B[k slot c][n] = C[2 c + ks][n]
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int kk = 2 * (lane & 3) + ks, nn = lane >> 2;
      cfp[ks] = (kk < N1 && nn < N1) ? chol_s[kk * N1 + nn] : 0.0;
    }
    int nu0 = 0, nucnt = 0;   // this warp's norm units
    {
      constexpr WsUnitTable<NCW> UT = ws_unit_table<NCW, NRT, KS, NEG, E * M>();
#pragma unroll
      for (int w = 0; w < NCW; ++w)
        if (warp == w) {
          nu0 = UT.first[w];
          nucnt = UT.cnt[w];
        }
    }
    // Gram-form norm item of this warp: R row tile grt x element group geg
    static_assert(C::LAG == 1, "the Gram / direct norm schedule assumes LAG = 1");
    const int gi = NCW - 1 - warp;
    const bool has_gi = gi >= 0 && gi < C::NGI;
    const int grt = has_gi ? gi / NEG : 0, geg = has_gi ? gi - (gi / NEG) * NEG : 0;
    double Rf[GRAM ? KS : 1];
    if constexpr (GRAM) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int row = grt * 8 + (lane >> 2), col = 4 * ks + (lane & 3);
        Rf[ks] = (gram && has_gi && row < KC) ? __ldg(a.gram_R + row * KC + col) : 0.0;
      }
    }
    // tile it-1 took the direct norm (its delta is in d_s); always, without GRAM
    int prev_direct = GRAM ? 0 : 1;
    for (int it = 0; it < n_my; ++it) {
      const int stage = it % NS;
      const int ob = it & 1;
      V3_T0(tc);
      WS_STAMP(warp, it, 0);
      mbar_wait(&qready_bar[stage], (it / NS) & 1);
      WS_STAMP(warp, it, 1);
      V3_ACC(3, tc);
      const int fast = mfast_s[stage];
      const bool gtile = GRAM && gram && fast;   // tile it: Gram-form norm
      const double* sst = sm + stage * C::STAGE;
      const double* ust = sst + TILE;
      const double* qst = ust + TILE + C::HALO;
      // direct norm of the previous tile (needs every warp's delta of tile it-1)
      double nprev = 0.0;
      if (it >= 1 && (!GRAM || prev_direct)) {
        const int jn = it - 1;
        V3_T0(td);
        mbar_wait(&done_bar[jn & 1], (jn >> 1) & 1);
        V3_ACC(8, td);
        WS_STAMP(warp, it, 2);
        V3_T0(tn);
        nprev = norm_units_swz<N1, M, E, UPW, C::DUE, C::DUC>(d_s + (jn % C::NDB) * C::DT, nu0, nucnt, lane, cfr,
                                                                   cfp, a.comp_w);
        V3_ACC(7, tn);
      }
      WS_STAMP(warp, it, 3);
      V3_T0(tm);
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
      const double* qb = qst + (lane >> 2) * KC + (lane & 3);
      WS_STAMP(warp, it, 4);
      if (fast && !IHDG_MEMONLY_ON) {
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
      } else if (!IHDG_MEMONLY_ON) {
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
      // Gram-form norm of tile it: Y = R dq for this warp's item, ||Y||_F^2
      // (comp_w and the reference mass are inside R, the Jacobian is applied
      // with the tile partial)
      double ng = 0.0;
      if constexpr (GRAM) {
        if (gtile && has_gi) {
          const double* dqb = qst + C::QT + (lane >> 2) * KC + (lane & 3) + geg * 8 * KC;
          double y0 = 0.0, y1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks)
            if (ks >= 2 * grt) dmma_8x8x4(y0, y1, Rf[ks], dqb[4 * ks]);
          ng = fma(y0, y0, y1 * y1);
        }
      }
      V3_ACC(4, tm);
      WS_STAMP(warp, it, 5);
      // a direct tile rewrites the d_s slot of tile it-2: every warp finished
      // that tile's norm by done(it-1)
      if (GRAM && !gtile && it >= 1 && !prev_direct) mbar_wait(&done_bar[(it - 1) & 1], ((it - 1) >> 1) & 1);
      V3_T0(to);
      if (it >= 2) mbar_wait(&outfree_bar[ob], ((it - 2) >> 1) & 1);
      V3_ACC(5, to);
      WS_STAMP(warp, it, 6);
      V3_T0(te);
      double* outb = out_s + ob * TILE;
      double* dcur = d_s + (it % C::NDB) * C::DT;
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
              if (!gtile) dcur[t * C::DUE + doff[j]] = acc[eg][j][v] - ust[t * NV + row];
            }
          }
        }
      }
      V3_ACC(10, te);
      WS_STAMP(warp, it, 7);
      if (it >= 1 && (!GRAM || prev_direct)) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nprev += __shfl_xor_sync(0xffffffffu, nprev, o);
        if (lane == 0) red_s[((it - 1) % C::NRED) * 32 + warp] = nprev;
      }
      if (GRAM && gtile) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ng += __shfl_xor_sync(0xffffffffu, ng, o);
        if (lane == 0) red_s[(it % C::NRED) * 32 + warp] = ng;
      }
      WS_STAMP(warp, it, 8);
      fence_proxy_async();
      __syncwarp();
      WS_STAMP(warp, it, 9);
      if (lane == 0) {
        mbar_arrive(&empty_bar[stage]);
        mbar_arrive(&done_bar[ob]);
      }
      if constexpr (GRAM) prev_direct = gtile ? 0 : 1;
    }
    // drain: direct norm of the last tile
    if (n_my >= 1 && (!GRAM || prev_direct)) {
      const int jn = n_my - 1;
      mbar_wait(&done_bar[jn & 1], (jn >> 1) & 1);
      double nsum = norm_units_swz<N1, M, E, UPW, C::DUE, C::DUC>(d_s + (jn % C::NDB) * C::DT, nu0, nucnt, lane, cfr,
                                                                       cfp, a.comp_w);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, o);
      if (lane == 0) red_s[(jn % C::NRED) * 32 + warp] = nsum;
    }
  }

  __syncthreads();
  if (tid == 0) {
    // the last LAG tiles (the prep warp wrote the partials before them)
    for (int jn = n_my - C::LAG > 0 ? n_my - C::LAG : 0; jn < n_my; ++jn) {
      if (jn <= n_my - 1 - C::LAG) continue;
      double s = 0.0;
      for (int w = 0; w < NCW; ++w) s += red_s[(jn % C::NRED) * 32 + w];
      a.tile_partials[blockIdx.x + jn * gridDim.x] = a.jac * s;
    }
  }
#ifdef IHDG_WS_PROF
  if (tid == 0) V3_ACC(6, tk0);
  V3_FLUSH;
#endif
  if (a.finalize) {
#ifndef IHDG_WS_SIMPLE_FIN
    if (a.layer_sums != nullptr && a.grid_bar != nullptr) {
      // Parallel finalize (launched cooperatively: every CTA is resident).
      // Phase 1: grid barrier on grid_bar once every tile partial is
      // written; phase 2: CTA b reduces the rows b, b + grid, ... (warp_row_sum,
      // one warp per row) into layer_sums; phase 3: the last CTA (ticket) sums
      // the layer sums in the fixed order -- bit-identical to finalize_block
      // over the tile partials.
      int64_t n_rows, row_len;
      partial_rows(geo, n_rows, row_len);
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        volatile unsigned* bar = a.grid_bar;
        const unsigned gen = bar[1];
        if (atomicAdd(a.grid_bar, 1u) == gridDim.x - 1) {
          a.grid_bar[0] = 0u;
          __threadfence();
          atomicAdd(a.grid_bar + 1, 1u);      // release the barrier (generation)
        } else {
          while (bar[1] == gen) __nanosleep(64);
        }
        __threadfence();
      }
      __syncthreads();
      const int nw = blockDim.x >> 5;
      for (int64_t r = (int64_t)blockIdx.x * nw + warp; r < n_rows; r += (int64_t)gridDim.x * nw) {
        const double rs = warp_row_sum(a.tile_partials + r * row_len, row_len, lane);
        if (lane == 0) a.layer_sums[r] = rs;
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        const unsigned tk = atomicAdd(&st->ticket, 1u);
        last_s = (tk == gridDim.x - 1);
      }
      __syncthreads();
      if (last_s) {
        __threadfence();
        finalize_block<1>(a.layer_sums, n_rows, 1, st, a.norm_hist);
      }
      return;
    }
#endif
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
      finalize_block<1>(a.tile_partials, n_rows, row_len, st, a.norm_hist);
    }
  }
}

}  // namespace ihdg
