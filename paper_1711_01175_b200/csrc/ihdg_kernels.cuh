// Generic iHDG-II kernels (any instantiated dim / order / ncomp).
//
// K2+K3  k_sweep        : fused gather -> lifted local solve -> write -> norm
// K4     k_class_apply  : per-element class operator (s = A^-1 b, s = P u^m)
// finalize_block        : fixed-order reduction of tile partials + stop rule
#pragma once

#include "ihdg_common.cuh"

namespace ihdg {

constexpr long long NO_NBR = -(1LL << 62);

// Sum of one row of tile partials by one warp: lane j sums the entries
// j, j+32, ... in order, then an xor butterfly (every lane ends with the same
// value: each stage adds a commutative pair).  Coalesced; the same code in
// k_layer_sums gives a rank's layer sums bit-identically.
__device__ __forceinline__ double warp_row_sum(const double* row, int64_t len, int lane) {
  double s = 0.0;
  for (int64_t i = lane; i < len; i += 32) s += __ldcg(row + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// Fixed-order, partition-independent sum of tile partials laid out as rows
// (one row per element layer of the slowest axis, row_len tiles each, in
// tile order; a strip partition splits between rows, never inside one):
// each row is summed by warp_row_sum, virtual lane v of 256 sums the row sums
// v, v+256, ... in order, then a fixed binary tree -- an order independent of
// the CTA size.  A rank's layer sums (k_layer_sums) therefore combine to
// exactly the single-rank value (ihdg_finalize with row_len 1: a one-entry
// row sums to itself).  Every thread of the CTA must call it; blockDim.x is a
// multiple of 32.
// RB virtual lanes of one warp are walked together (independent loads in
// flight); any RB gives the same value.  Small RB keeps the code small where
// the reduction is off the hot path's instruction cache footprint (k_sweep_ws).
template <int RB = 8>
__device__ inline double rows_sum(const double* parts, int64_t n_rows, int64_t row_len) {
  __shared__ double red[256];
  __syncthreads();
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (row_len == 1) {
    // one-entry rows (layer sums): warp_row_sum of a row is the entry itself
    // (the butterfly only adds zeros), so one thread per virtual lane adds
    // its rows v, v + 256, ... in order -- the same value bit for bit, without
    // a dependent load and five shuffles per row
    for (int v = threadIdx.x; v < 256; v += blockDim.x) {
      double s = 0.0;
      for (int64_t r0 = v; r0 < n_rows; r0 += 256 * 8) {
        double x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int64_t r = r0 + 256 * (int64_t)j;
          x[j] = r < n_rows ? __ldcg(parts + r) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (r0 + 256 * (int64_t)j < n_rows) s += x[j];
      }
      red[v] = s;
    }
  } else {
    // a warp takes RB virtual lanes at a time (v = vb + j nw) and walks their
    // rows v, v + 256, ... together: RB independent row loads in flight, each
    // row still summed by warp_row_sum's per-lane order and butterfly and each
    // virtual lane still adding its rows in order -- the same bits for any RB
    for (int vb = threadIdx.x >> 5; vb < 256; vb += nw * RB) {
      double s[RB];
#pragma unroll
      for (int j = 0; j < RB; ++j) s[j] = 0.0;
      for (int64_t k = 0; 256 * k < n_rows; ++k) {
        double rs[RB];
#pragma unroll
        for (int j = 0; j < RB; ++j) rs[j] = 0.0;
        for (int64_t i = lane; i < row_len; i += 32) {
          double x[RB];
#pragma unroll
          for (int j = 0; j < RB; ++j) {
            const int v = vb + j * nw;
            const int64_t r = v + 256 * k;
            x[j] = (v < 256 && r < n_rows) ? __ldcg(parts + r * row_len + i) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < RB; ++j) rs[j] += x[j];
        }
#pragma unroll
        for (int j = 0; j < RB; ++j) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) rs[j] += __shfl_xor_sync(0xffffffffu, rs[j], o);
          if (vb + j * nw + 256 * k < n_rows) s[j] += rs[j];
        }
      }
#pragma unroll
      for (int j = 0; j < RB; ++j)
        if (lane == 0 && vb + j * nw < 256) red[vb + j * nw] = s[j];
    }
  }
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    for (int v = threadIdx.x; v < w; v += blockDim.x) red[v] += red[v + w];
    __syncthreads();
  }
  return red[0];
}

// rows of the tile partials of a strip (see rows_sum): one per layer in 2D /
// 3D, the whole strip in 1D
__host__ __device__ inline void partial_rows(const Geo& g, int64_t& n_rows, int64_t& row_len) {
  n_rows = g.D == 1 ? 1 : g.nlay;
  row_len = g.D == 1 ? g.ntiles : g.segs;
}

// The stopping / divergence logic of `run` (
// PAPER.md:1308-1311) on the fixed-order sum of the partials.  Must be
// executed by every thread of one CTA.
template <int RB = 8>
__device__ inline void finalize_block(const double* parts, int64_t n_rows, int64_t row_len, ihdg_iter_state* st,
                                      double* hist) {
  const double total = rows_sum<RB>(parts, n_rows, row_len);
  if (threadIdx.x == 0) {
    const double norm = sqrt(total);
    const int it = st->iters + 1;
    st->iters = it;
    if (hist != nullptr && it <= st->max_iters) hist[it - 1] = norm;
    if (it == 1) st->first_norm = norm;
    st->last_norm = norm;
    int status = IHDG_RUNNING;
    if (!(norm == norm)) status = IHDG_NAN;
    else if (norm < st->tol) status = IHDG_CONVERGED;
    else if (it > 1 && norm > st->diverge_factor * st->first_norm) status = IHDG_DIVERGED;
    else if (it >= st->max_iters) status = IHDG_MAXITER;
    st->status = status;
    st->ticket = 0u;
    __threadfence();
  }
}

template <int D, int N1, int M>
struct SweepSmem {
  using C = Cfg<D, N1, M>;
  // q: up to 4 raw blocks per face node (per-element operators, iHDG-I)
  static constexpr size_t doubles = 4 * (size_t)C::KIN * C::TE + 2 * (size_t)C::TE * C::NV +
                                    N1 * N1 + C::TE * (2 * D + 1);
  static constexpr size_t bytes = doubles * sizeof(double);
};

// One iHDG-II sweep (Algorithm 1 lines 2-4) over a strip.
// Each CTA walks tiles of TE consecutive elements of one layer:
//   1. neighbour ids + boundary mask -> operator class
//   2. q[k][t]: neighbour iterate-k face scalars (TraceSnapshot)
//   3. u^{k+1} = s + L_class q  (apply_local in lifted form),
//      threads own rows, L is read once per tile and reused over TE elements
//   4. delta = u^{k+1} - u^k; mass-weighted (sum-factorised Cholesky of the
//      1D mass) or trace norm -> one partial per tile in a fixed order.
template <int D, int N1, int M>
__global__ void __launch_bounds__(Cfg<D, N1, M>::NT)
    k_sweep(const ihdg_sweep_args a) {
  using C = Cfg<D, N1, M>;
  constexpr int NP = C::NP, NV = C::NV, NF = C::NF, KIN = C::KIN;
  constexpr int TE = C::TE, RP = C::RP, G = C::G, NT = C::NT, J = C::J;
  constexpr int NFACE = 2 * D;

  extern __shared__ __align__(16) double sm[];
  // per-element operators with raw neighbour values (ihdg.h): kin columns
  const int rb = a.raw_blocks > 0 ? a.raw_blocks : 1;
  const int kin = KIN * rb;
  double* q_s = sm;                 // [kin][TE]
  double* d_s = q_s + 4 * KIN * TE; // [TE][NV]
  double* t_s = d_s + TE * NV;      // [TE][NV]
  double* c_s = t_s + TE * NV;      // [N1][N1]
  double* pf_s = c_s + N1 * N1;     // [TE][NFACE+1]
  __shared__ int fv_s[NFACE][NF];
  __shared__ int cls_s[TE];
  __shared__ long long nb_s[TE][NFACE];
  __shared__ int uni_s;
  __shared__ int last_s;

  ihdg_iter_state* st = a.state;
  if (st->status != IHDG_RUNNING) return;

  Geo geo;
  geo.init(a.g, TE);
  const int tid = threadIdx.x;
  for (int i = tid; i < NFACE * NF; i += NT) fv_s[i / NF][i % NF] = face_node_vidx(D, N1, i / NF, i % NF);
  for (int i = tid; i < N1 * N1; i += NT) c_s[i] = a.chol1d[i];

  const int64_t ls = geo.ls;
  const double* __restrict__ uo = a.u_old + ls * NV;
  double* __restrict__ un = a.u_new + ls * NV;
  const double* __restrict__ sv = a.s;

  for (int64_t tile = blockIdx.x; tile < geo.ntiles; tile += gridDim.x) {
    int64_t e0;
    int nt;
    geo.tile_range(tile, TE, e0, nt);
    __syncthreads();
    if (tid < TE) {
      const int t = tid;
      if (t < nt) {
        const int64_t e = e0 + t;
        int64_t idx[3];
        geo.multi_index(e, idx);
        int mask = 0;
        for (int f = 0; f < NFACE; ++f) {
          int64_t nb;
          if (geo.neighbor(e, idx, f, nb)) {
            nb_s[t][f] = nb;
          } else {
            nb_s[t][f] = NO_NBR;
            mask |= 1 << f;
          }
        }
        cls_s[t] = a.per_element ? (int)e : a.class_of_mask[mask];
      } else {
        cls_s[t] = -1;
      }
    }
    __syncthreads();
    if (tid == 0) {
      int u = !a.per_element;
      for (int t = 1; t < nt; ++t) u &= (cls_s[t] == cls_s[0]);
      uni_s = u;
    }
    // -- gather neighbour face scalars (iterate k) --------------------------
    if (a.raw_blocks > 0) {
      // raw face-node values (per-element operators): column (f, j, n)
      for (int i = tid; i < kin * TE; i += NT) {
        const int k = i / TE, t = i % TE;
        const int f = k / (rb * NF), j = (k / NF) % rb, n = k % NF;
        double v = 0.0;
        if (t < nt) {
          const int c = a.raw_comp[f][j];
          if (j < 2) {
            const long long nb = nb_s[t][f];
            if (nb != NO_NBR && a.coupled[f]) v = __ldg(uo + nb * NV + c * NP + fv_s[f ^ 1][n]);
          } else {
            v = __ldg(uo + (e0 + t) * NV + c * NP + fv_s[f][n]);
          }
        }
        q_s[i] = v;
      }
    } else
    for (int i = tid; i < KIN * TE; i += NT) {
      const int k = i / TE, t = i % TE;
      const int f = k / NF, n = k % NF;
      double v = 0.0;
      if (t < nt && a.coupled[f]) {
        const long long nb = nb_s[t][f];
        if (nb != NO_NBR) {
          const double* p = uo + nb * NV + fv_s[f ^ 1][n];
#pragma unroll
          for (int c = 0; c < M; ++c) v = fma(a.face_w[f][c], __ldg(p + c * NP), v);
        }
        if (a.scheme == IHDG_SCHEME_I) {
          // iHDG-I: the element's own iterate-k face scalar joins the trace
          const double* po = uo + (e0 + t) * NV + fv_s[f][n];
#pragma unroll
          for (int c = 0; c < M; ++c) v = fma(a.own_w[f][c], __ldg(po + c * NP), v);
        }
      }
      q_s[i] = v;
    }
    __syncthreads();
    // -- lifted local solve: rows x elements --------------------------------
    const int r = tid % RP, gi = tid / RP;
    for (int r0 = 0; r0 < NV; r0 += RP) {
      const int rr = r0 + r;
      const bool rv = rr < NV;
      double acc[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int t = gi + j * G;
        acc[j] = (rv && t < nt) ? __ldg(sv + (e0 + t) * NV + rr) : 0.0;
      }
      if (uni_s) {
        const double* __restrict__ Lc = a.LT + (size_t)cls_s[0] * KIN * NV + (rv ? rr : 0);
#pragma unroll 4
        for (int k = 0; k < KIN; ++k) {
          const double l = __ldg(Lc + (size_t)k * NV);
#pragma unroll
          for (int j = 0; j < J; ++j) acc[j] = fma(l, q_s[k * TE + gi + j * G], acc[j]);
        }
      } else if (rv) {
        // per element (mixed classes at the boundary; every element its own
        // operator in GEMV mode: a memory-bound stream of L)
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const int t = gi + j * G;
          if (t < nt) {
            const double* __restrict__ Lc = a.LT + (size_t)cls_s[t] * kin * NV + rr;
            double s = acc[j];
#pragma unroll 4
            for (int k = 0; k < kin; ++k) s = fma(__ldg(Lc + (size_t)k * NV), q_s[k * TE + t], s);
            acc[j] = s;
          }
        }
      }
      if (rv) {
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const int t = gi + j * G;
          if (t < nt) {
            const int64_t o = (e0 + t) * NV + rr;
            un[o] = acc[j];
            d_s[t * NV + rr] = acc[j] - __ldg(uo + o);
          }
        }
      }
    }
    __syncthreads();
    // -- stopping norm of the successive difference --------------------------
    if (a.norm_kind == IHDG_NORM_VOLUME) {
      // ||delta||_M^2 = J * sum_c w_c |(C^T (x) ... (x) C^T) delta_c|^2
      double* src = d_s;
      double* dst = t_s;
      int mul = 1;
      for (int ax = 0; ax < D; ++ax) {
        for (int i = tid; i < nt * NV; i += NT) {
          const int t = i / NV, rem = i % NV;
          const int n = rem % NP;
          const int ia = (n / mul) % N1;
          const int base = t * NV + rem - ia * mul;
          double v = 0.0;
          for (int ip = ia; ip < N1; ++ip) v = fma(c_s[ip * N1 + ia], src[base + ip * mul], v);
          dst[i] = v;
        }
        __syncthreads();
        double* tmp = src;
        src = dst;
        dst = tmp;
        mul *= N1;
      }
      const int warp = tid >> 5, lane = tid & 31;
      for (int t = warp; t < nt; t += NT / 32) {
        double s = 0.0;
        for (int i = lane; i < NV; i += 32) {
          const double v = src[t * NV + i];
          s = fma(a.comp_w[i / NP] * v, v, s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) pf_s[t * (NFACE + 1)] = a.jac * s;
      }
    } else {
      // skeleton L2 norm of the trace update on the flagged (outflow) faces
      for (int i = tid; i < nt * NFACE; i += NT) {
        const int t = i / NFACE, f = i % NFACE;
        double v = 0.0;
        if (a.out_face[f]) {
          double x[NF], y[NF];
#pragma unroll
          for (int n = 0; n < NF; ++n) {
            double w = 0.0;
#pragma unroll
            for (int c = 0; c < M; ++c) w = fma(a.out_w[f][c], d_s[t * NV + c * NP + fv_s[f][n]], w);
            x[n] = w;
          }
          int mul = 1;
#pragma unroll
          for (int ax = 0; ax < D - 1; ++ax) {
#pragma unroll
            for (int n = 0; n < NF; ++n) {
              const int ia = (n / mul) % N1;
              double w = 0.0;
              for (int ip = ia; ip < N1; ++ip) w = fma(c_s[ip * N1 + ia], x[n + (ip - ia) * mul], w);
              y[n] = w;
            }
#pragma unroll
            for (int n = 0; n < NF; ++n) x[n] = y[n];
            mul *= N1;
          }
#pragma unroll
          for (int n = 0; n < NF; ++n) v = fma(x[n], x[n], v);
          v *= a.jac_face[f >> 1];
        }
        pf_s[t * (NFACE + 1) + 1 + f] = v;
      }
      __syncthreads();
      if (tid < nt) {
        double s = 0.0;
        for (int f = 0; f < NFACE; ++f) s += pf_s[tid * (NFACE + 1) + 1 + f];
        pf_s[tid * (NFACE + 1)] = s;
      }
    }
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int t = 0; t < nt; ++t) s += pf_s[t * (NFACE + 1)];
      a.tile_partials[tile] = s;
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

template <int D, int N1, int M>
struct ApplySmem {
  using C = Cfg<D, N1, M>;
  static constexpr size_t bytes = (size_t)C::NV * C::TE * sizeof(double);
};

// out[e][r] (+)= sum_k opT[class(e)][k][r] * in[e][in_offset + k]
template <int D, int N1, int M>
__global__ void __launch_bounds__(Cfg<D, N1, M>::NT)
    k_class_apply(const ihdg_class_apply_args a) {
  using C = Cfg<D, N1, M>;
  constexpr int NV = C::NV, TE = C::TE, RP = C::RP, G = C::G, NT = C::NT, J = C::J;
  constexpr int NFACE = 2 * D;
  extern __shared__ __align__(16) double sm[];
  double* in_s = sm;  // [ncols][TE]
  __shared__ int cls_s[TE];
  __shared__ int uni_s;
  Geo geo;
  geo.init(a.g, TE);
  const int tid = threadIdx.x;
  const int ncols = a.ncols;
  const double* in0 = a.in + (a.in_ghost ? geo.ls * a.in_stride : 0) + a.in_offset;
  double* out0 = a.out + (a.out_ghost ? geo.ls * NV : 0);
  for (int64_t tile = blockIdx.x; tile < geo.ntiles; tile += gridDim.x) {
    int64_t e0;
    int nt;
    geo.tile_range(tile, TE, e0, nt);
    __syncthreads();
    if (tid < TE) {
      const int t = tid;
      if (t < nt) {
        const int64_t e = e0 + t;
        int64_t idx[3];
        geo.multi_index(e, idx);
        int mask = 0;
        for (int f = 0; f < NFACE; ++f) {
          int64_t nb;
          if (!geo.neighbor(e, idx, f, nb)) mask |= 1 << f;
        }
        cls_s[t] = a.per_element ? (int)e : a.class_of_mask[mask];
      } else {
        cls_s[t] = -1;
      }
    }
    for (int i = tid; i < ncols * TE; i += NT) {
      const int k = i / TE, t = i % TE;
      in_s[i] = (t < nt) ? in0[(e0 + t) * a.in_stride + k] : 0.0;
    }
    __syncthreads();
    if (tid == 0) {
      int u = !a.per_element;
      for (int t = 1; t < nt; ++t) u &= (cls_s[t] == cls_s[0]);
      uni_s = u;
    }
    __syncthreads();
    const int r = tid % RP, gi = tid / RP;
    for (int r0 = 0; r0 < NV; r0 += RP) {
      const int rr = r0 + r;
      if (rr >= NV) continue;
      double acc[J];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int t = gi + j * G;
        acc[j] = (a.accumulate && t < nt) ? out0[(e0 + t) * NV + rr] : 0.0;
      }
      if (uni_s) {
        const double* Op = a.opT + (size_t)cls_s[0] * ncols * NV + rr;
        for (int k = 0; k < ncols; ++k) {
          const double l = __ldg(Op + (size_t)k * NV);
#pragma unroll
          for (int j = 0; j < J; ++j) acc[j] = fma(l, in_s[k * TE + gi + j * G], acc[j]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < J; ++j) {
          const int t = gi + j * G;
          if (t < nt) {
            const double* Op = a.opT + (size_t)cls_s[t] * ncols * NV + rr;
            double s = acc[j];
            for (int k = 0; k < ncols; ++k) s = fma(__ldg(Op + (size_t)k * NV), in_s[k * TE + t], s);
            acc[j] = s;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const int t = gi + j * G;
        if (t < nt) out0[(e0 + t) * NV + rr] = acc[j];
      }
    }
  }
}

}  // namespace ihdg
