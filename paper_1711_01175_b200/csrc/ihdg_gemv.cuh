// iHDG sweep with per-element operators (the GEMV mode of BASELINE.json's
// north_star: "a batched small dense GEMV, memory-bound, when local operators
// differ per element"; ihdg.h: per_element = 1, raw_blocks = 2 or 4).
//
// Every element streams its own L_e = A_e^-1 B_e (LT_e: kin x NV doubles, 93 KB
// for 3D p=2) exactly once per sweep, so the kernel is a bandwidth pump:
//
//   producer warp  : TMA bulk copies (cp.async.bulk) of LT_e in chunks of CH
//                    columns (~24 KB, contiguous in memory) into an NS-stage
//                    shared-memory ring, across element and tile boundaries
//                    (full / empty mbarriers);
//   consumer warps : thread = row of L_e.  q_e (raw neighbour face-node values
//                    of iterate k, TraceSnapshot) is gathered one element
//                    ahead into registers together with s_e and u^k_e, so the
//                    only wait in the element loop is on the ring;
//                    u^{k+1} = s + L_e q as one FMA chain per row in column
//                    order (the generic kernel's order: same bits), stored
//                    from registers; delta -> the mass-weighted norm by
//                    sum-factorised Cholesky passes in shared memory.
//
// One CTA owns one tile (the generic kernel's TE consecutive elements: one
// tile partial, summed over its elements in order), several CTAs per SM; the
// grid is min(tiles, resident CTAs), so on meshes of a few hundred tiles every
// tile streams concurrently and the shared HBM balances them.
//
// HBM per element-DOF: 8 (kin + 3) B (L_e, s, u^k, u^{k+1}).
#pragma once

#include <climits>

#include "ihdg_stream.cuh"

namespace ihdg {

template <int D, int N1, int M>
struct GCfg {
  using C = Cfg<D, N1, M>;
  static constexpr int NP = C::NP, NV = C::NV, NF = C::NF, NFACE = 2 * D, KIN = C::KIN;
  static constexpr int TE = C::TE;                  // elements per tile (= the generic kernel's: one partial)
  static constexpr int NCW = (NV + 31) / 32;        // consumer warps (thread = row)
  static constexpr int NCT = 32 * NCW;
  static constexpr int NT = NCT + 32;               // + producer warp
  static constexpr int KMAX = 4 * KIN;              // raw_blocks <= 4
  // columns per chunk: about 24 KB, even (16-byte multiples for odd NV)
#ifndef IHDG_GEMV_CHB
#define IHDG_GEMV_CHB 24576   // chunk bytes (A/B: 8 / 12 / 16 / 24 / 32 / 48 KB; 24 KB x 3 stages measured best)
#endif
  static constexpr int CH0 = IHDG_GEMV_CHB / (NV * 8);
  static constexpr int CH = CH0 < 2 ? 2 : (CH0 > 64 ? 64 : CH0 / 2 * 2);
#ifndef IHDG_GEMV_NS
#define IHDG_GEMV_NS 3
#endif
  static constexpr int NS = IHDG_GEMV_NS;           // ring stages
  static constexpr int STAGE = CH * NV;             // doubles
  static constexpr int QM = (KMAX + NCT - 1) / NCT; // gathered q entries per consumer thread
  static constexpr int OFF_Q = NS * STAGE;          // q[2][KMAX]
  static constexpr int OFF_D = OFF_Q + 2 * KMAX;    // delta / pass buffers [2][NV]
  static constexpr int N_DBL = OFF_D + 2 * NV + N1 * N1;
  static constexpr size_t BYTES = (size_t)N_DBL * sizeof(double) + 2 * NS * sizeof(uint64_t);
  static_assert((STAGE * sizeof(double)) % 16 == 0, "chunk bytes must be 16-byte multiples");
  static_assert(BYTES + 2048 <= 232448, "shared memory over the sm_100a opt-in limit");
};

template <int D, int N1, int M>
__global__ void __launch_bounds__(GCfg<D, N1, M>::NT) k_sweep_gemv(const ihdg_sweep_args a) {
  using G = GCfg<D, N1, M>;
  constexpr int NP = G::NP, NV = G::NV, NF = G::NF, NFACE = G::NFACE, KIN = G::KIN;
  constexpr int TE = G::TE, NCW = G::NCW, NCT = G::NCT, CH = G::CH, NS = G::NS, QM = G::QM;

  extern __shared__ __align__(16) double sm[];
  double* q_s = sm + G::OFF_Q;
  double* d_s = sm + G::OFF_D;
  double* t_s = d_s + NV;
  double* c_s = t_s + NV;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sm + G::N_DBL);
  uint64_t* empty_bar = full_bar + NS;
  __shared__ int fv_s[NFACE][NF];
  __shared__ int last_s;

  ihdg_iter_state* st = a.state;
  pdl_launch_dependents();   // the next launch may start its own prologue

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  Geo geo;
  geo.init(a.g, TE);
  const int rb = a.raw_blocks;
  const int kin = KIN * rb;
  const int nch = (kin + CH - 1) / CH;
  const int64_t ls = geo.ls;
  const double* __restrict__ uo = a.u_old + ls * NV;
  double* __restrict__ un = a.u_new + ls * NV;

  for (int i = tid; i < NFACE * NF; i += blockDim.x) fv_s[i / NF][i % NF] = face_node_vidx(D, N1, i / NF, i % NF);
  for (int i = tid; i < N1 * N1; i += blockDim.x) c_s[i] = a.chol1d[i];
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // everything above reads only launch-invariant data; the operators' stream,
  // the iterate and the iteration state wait for the previous launches
  pdl_wait();
  if (st->status != IHDG_RUNNING) return;

  if (warp == NCW) {
    // ============================ producer warp ============================
    if (lane == 0) {
      int cnt = 0;
      for (int64_t tile = blockIdx.x; tile < geo.ntiles; tile += gridDim.x) {
        int64_t e0;
        int nt;
        geo.tile_range(tile, TE, e0, nt);
        for (int t = 0; t < nt; ++t) {
          const double* Le = a.LT + (size_t)(e0 + t) * kin * NV;
          for (int c = 0; c < nch; ++c, ++cnt) {
            const int stage = cnt % NS;
            if (cnt >= NS) mbar_wait(&empty_bar[stage], ((cnt / NS) - 1) & 1);
            const int cols = (kin - c * CH) < CH ? (kin - c * CH) : CH;
            const uint32_t bytes = (uint32_t)(cols * NV * sizeof(double));
            mbar_arrive_expect_tx(&full_bar[stage], bytes);
            bulk_g2s(sm + stage * G::STAGE, Le + (size_t)c * CH * NV, bytes, &full_bar[stage]);
          }
        }
      }
    }
  } else {
    // ============================ consumer warps ===========================
    const int row = tid;
    const bool rv = row < NV;
    // 32-bit element geometry (the dispatch guarantees local counts < 2^31):
    // multi-index by two FastDiv divisions per element, neighbours as in
    // Geo::neighbor (ghost layers beyond the strip on the last axis)
    const int c0 = (int)geo.c[0], c1 = (int)geo.c[1];
    const int lsi = (int)ls, nlay = (int)geo.nlay, lb = (int)geo.lb;
    FastDiv dc0, dc1;
    dc0.init((uint32_t)c0);
    dc1.init((uint32_t)c1);
    constexpr int NONE = INT_MIN;
    auto neighbour = [&](int e, int f) -> int {
      int idx[3];
      const int r = dc0.div(e);
      idx[0] = e - r * c0;
      if (D == 3) {
        const int l = dc1.div(r);
        idx[1] = r - l * c1;
        idx[2] = lb + l;
      } else {
        idx[1] = lb + r;
        idx[2] = 0;
      }
      const int ax = f >> 1, sd = f & 1;
      const int cn = (int)geo.c[ax];
      int j = idx[ax] + (sd ? 1 : -1);
      if (j < 0) {
        if (!geo.per[ax]) return NONE;
        j = cn - 1;
      } else if (j >= cn) {
        if (!geo.per[ax]) return NONE;
        j = 0;
      }
      if (ax < D - 1) return e + (j - idx[ax]) * (ax == 0 ? 1 : c0);
      const int lay = idx[D - 1] - lb, in_layer = e - lay * lsi;
      const int l = j - lb;
      return ((l >= 0 && l < nlay) ? l : (sd ? nlay : -1)) * lsi + in_layer;
    };
    // gather of one q entry: raw face-node value of the neighbour across face
    // f (blocks 0, 1) or of the element itself (blocks 2, 3: iHDG-I)
    auto gather = [&](int e, int k) -> double {
      const int f = k / (rb * NF), j = (k / NF) % rb, n = k % NF;
      const int c = a.raw_comp[f][j];
      if (j >= 2) return __ldg(uo + (int64_t)e * NV + c * NP + fv_s[f][n]);
      if (!a.coupled[f]) return 0.0;
      const int nb = neighbour(e, f);
      if (nb == NONE) return 0.0;
      return __ldg(uo + (int64_t)nb * NV + c * NP + fv_s[f ^ 1][n]);
    };
    // operands of one element, loaded one element ahead
    double qn[QM], sn = 0.0, ukn = 0.0;
    auto prefetch = [&](int e) {
#pragma unroll
      for (int m = 0; m < QM; ++m) {
        const int k = tid + m * NCT;
        qn[m] = k < kin ? gather(e, k) : 0.0;
      }
      sn = rv ? __ldg(a.s + (int64_t)e * NV + row) : 0.0;
      ukn = rv ? __ldg(uo + (int64_t)e * NV + row) : 0.0;
    };
    int cnt = 0, cur = 0;
    bool first = true;
    for (int64_t tile = blockIdx.x; tile < geo.ntiles; tile += gridDim.x) {
      int64_t e0;
      int nt;
      geo.tile_range(tile, TE, e0, nt);
      if (first) {
        prefetch((int)e0);
        first = false;
      }
      double tile_sum = 0.0;   // warp 0, lane 0: the tile partial, its elements in order
      for (int t = 0; t < nt; ++t) {
        const int64_t e = e0 + t;
        // this element's operands (prefetched) -> q to shared memory
        double* qc = q_s + cur * G::KMAX;
#pragma unroll
        for (int m = 0; m < QM; ++m) {
          const int k = tid + m * NCT;
          if (k < kin) qc[k] = qn[m];
        }
        double acc = sn;
        const double uk = ukn;
        named_bar_sync(1, NCT);   // q visible; the previous element's norm reads of d_s / t_s are done
        // next element of this CTA (next tile's first element at a tile end)
        {
          int64_t en = -1;
          if (t + 1 < nt) {
            en = e + 1;
          } else if (tile + gridDim.x < geo.ntiles) {
            int ntn;
            geo.tile_range(tile + gridDim.x, TE, en, ntn);
          }
          if (en >= 0) prefetch((int)en);
        }
        // stream L_e through the ring: one FMA chain per row, columns in order
        for (int c = 0; c < nch; ++c, ++cnt) {
          const int stage = cnt % NS;
          mbar_wait(&full_bar[stage], (cnt / NS) & 1);
          const double* Ls = sm + stage * G::STAGE + (rv ? row : 0);
          const double* qk = qc + c * CH;
          const int cols = (kin - c * CH) < CH ? (kin - c * CH) : CH;
          if (cols == CH) {
#pragma unroll
            for (int k = 0; k < CH; ++k) acc = fma(Ls[k * NV], qk[k], acc);
          } else {
            for (int k = 0; k < cols; ++k) acc = fma(Ls[k * NV], qk[k], acc);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty_bar[stage]);
        }
        if (rv) {
          un[e * NV + row] = acc;
          d_s[row] = acc - uk;
        }
        named_bar_sync(1, NCT);
        // ||delta||_M^2 = J sum_c w_c |(C^T x ... x C^T) delta_c|^2 (the generic kernel's passes)
        double* src = d_s;
        double* dst = t_s;
        int mul = 1;
#pragma unroll
        for (int ax = 0; ax < D; ++ax) {
          if (rv) {
            const int n = row % NP;
            const int ia = (n / mul) % N1;
            const int base = row - ia * mul;
            double v = 0.0;
            for (int ip = ia; ip < N1; ++ip) v = fma(c_s[ip * N1 + ia], src[base + ip * mul], v);
            dst[row] = v;
          }
          named_bar_sync(1, NCT);
          double* tmp = src;
          src = dst;
          dst = tmp;
          mul *= N1;
        }
        if (warp == 0) {
          double s = 0.0;
          for (int i = lane; i < NV; i += 32) {
            const double v = src[i];
            s = fma(a.comp_w[i / NP] * v, v, s);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          tile_sum = __dadd_rn(tile_sum, __dmul_rn(a.jac, s));   // product rounded first, as the generic kernel stores it
        }
        cur ^= 1;
      }
      if (tid == 0) a.tile_partials[tile] = tile_sum;
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
      int64_t n_rows, row_len;
      partial_rows(geo, n_rows, row_len);
      finalize_block(a.tile_partials, n_rows, row_len, st, a.norm_hist);
    }
  }
}

}  // namespace ihdg
