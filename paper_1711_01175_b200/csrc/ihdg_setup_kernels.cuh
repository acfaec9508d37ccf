// Setup kernels: K1 assembly + Gauss-Jordan inversion, analytic field
// evaluation, quadrature projection, trace extraction.
#pragma once

#include "ihdg_common.cuh"
#include "ihdg_kernels.cuh"

namespace ihdg {

// ---------------------------------------------------------------------------
// K1: Kronecker term-list assembly (one CTA per operator class).
// A local matrix of the substituted iHDG-II weak form (SPEC.md:246-274,
// PAPER.md:409-420, 714-727, 1067-1077) is a sum of tensor products of 1D
// reference matrices (mass, convection, endpoint projectors) times
// coefficients; the host (assembly.py) derives the term list, this kernel
// evaluates the entries in fp64.
// ---------------------------------------------------------------------------
struct AsmDims {
  int D, N1, NP, NV, NF, KIN, nr;
};

__global__ void k_assemble_build(const ihdg_assembly_args a, AsmDims dm) {
  const int cls = blockIdx.x;
  const int tid = threadIdx.x, nth = blockDim.x;
  double* A = a.A + (size_t)cls * dm.NV * dm.NV;
  double* B = a.B + (size_t)cls * dm.NV * dm.KIN;
  double* R = a.R ? a.R + (size_t)cls * dm.NV * dm.nr : nullptr;
  for (int i = tid; i < dm.NV * dm.NV; i += nth) A[i] = 0.0;
  for (int i = tid; i < dm.NV * dm.KIN; i += nth) B[i] = 0.0;
  if (R)
    for (int i = tid; i < dm.NV * dm.nr; i += nth) R[i] = 0.0;
  __syncthreads();
  const int N1 = dm.N1;
  for (int tm = 0; tm < a.n_terms; ++tm) {
    const int* T = a.terms + 8 * tm;
    if (T[0] != cls) continue;
    const int target = T[1], rc = T[2], cb = T[3];
    const double coef = a.coefs[tm];
    int nc[3] = {1, 1, 1};
    const double* op[3] = {nullptr, nullptr, nullptr};
    int ncols = 1;
    for (int ax = 0; ax < dm.D; ++ax) {
      op[ax] = a.ops1d + (size_t)T[4 + ax] * N1 * N1;
      nc[ax] = a.op_ncols[T[4 + ax]];
      ncols *= nc[ax];
    }
    double* dst;
    int ld, col0;
    if (target == 0) {
      dst = A; ld = dm.NV; col0 = cb * dm.NP;
    } else if (target == 1) {
      dst = B; ld = dm.KIN; col0 = cb * dm.NF;
    } else {
      dst = R; ld = dm.nr; col0 = cb * dm.NP;
    }
    if (dst == nullptr) continue;
    for (int idx = tid; idx < dm.NP * ncols; idx += nth) {
      int i = idx / ncols, j = idx % ncols;
      double v = coef;
      int ii = i, jj = j;
      for (int ax = 0; ax < dm.D; ++ax) {
        const int ia = ii % N1, ja = jj % nc[ax];
        ii /= N1;
        jj /= nc[ax];
        v *= op[ax][ia * N1 + ja];
      }
      dst[(size_t)(rc * dm.NP + i) * ld + col0 + j] += v;
    }
    __syncthreads();
  }
}

// In-place Gauss-Jordan inversion with partial pivoting (row swaps undone by
// column swaps in reverse), one CTA per class, matrix in global memory.
__global__ void k_gauss_jordan(const ihdg_assembly_args a, AsmDims dm, int* perm_ws) {
  const int cls = blockIdx.x;
  const int n = dm.NV;
  const int tid = threadIdx.x, nth = blockDim.x;
  double* M = a.Ainv + (size_t)cls * n * n;
  const double* A = a.A + (size_t)cls * n * n;
  int* perm = perm_ws + (size_t)cls * n;
  extern __shared__ double gj_s[];
  double* colk = gj_s;       // [n]
  double* rowk = gj_s + n;   // [n]
  __shared__ double bval[1024];
  __shared__ int bidx[1024];
  __shared__ double minpiv;
  for (int i = tid; i < n * n; i += nth) M[i] = A[i];
  if (tid == 0) minpiv = 1e300;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    // pivot search: max |M[i][k]|, i >= k, ties -> smallest i
    double bv = -1.0;
    int bi = n;
    for (int i = k + tid; i < n; i += nth) {
      const double v = fabs(M[(size_t)i * n + k]);
      if (v > bv) { bv = v; bi = i; }
    }
    bval[tid] = bv;
    bidx[tid] = bi;
    __syncthreads();
    for (int w = nth / 2; w > 0; w >>= 1) {
      if (tid < w) {
        const double v2 = bval[tid + w];
        const int i2 = bidx[tid + w];
        if (v2 > bval[tid] || (v2 == bval[tid] && i2 < bidx[tid])) {
          bval[tid] = v2;
          bidx[tid] = i2;
        }
      }
      __syncthreads();
    }
    const int p = bidx[0];
    if (tid == 0) {
      perm[k] = p;
      if (bval[0] < minpiv) minpiv = bval[0];
    }
    if (p != k) {
      for (int j = tid; j < n; j += nth) {
        const double t = M[(size_t)k * n + j];
        M[(size_t)k * n + j] = M[(size_t)p * n + j];
        M[(size_t)p * n + j] = t;
      }
    }
    __syncthreads();
    const double piv = M[(size_t)k * n + k];
    for (int j = tid; j < n; j += nth) {
      rowk[j] = (j == k ? 1.0 : M[(size_t)k * n + j]) / piv;
      colk[j] = M[(size_t)j * n + k];
    }
    __syncthreads();
    for (int idx = tid; idx < n * n; idx += nth) {
      const int i = idx / n, j = idx % n;
      if (i == k) {
        M[idx] = rowk[j];
      } else {
        const double base = (j == k) ? 0.0 : M[idx];
        M[idx] = fma(-colk[i], rowk[j], base);
      }
    }
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {
    const int p = perm[k];
    if (p != k) {
      for (int i = tid; i < n; i += nth) {
        const double t = M[(size_t)i * n + k];
        M[(size_t)i * n + k] = M[(size_t)i * n + p];
        M[(size_t)i * n + p] = t;
      }
    }
    __syncthreads();
  }
  if (tid == 0) a.min_pivot[cls] = minpiv;
}

// LT[c][k][r] = sum_j Ainv[r][j] B[j][k];  PT likewise with R;  AinvT.
__global__ void k_assemble_lift(const ihdg_assembly_args a, AsmDims dm) {
  const int cls = blockIdx.x;
  const int n = dm.NV;
  const double* Ai = a.Ainv + (size_t)cls * n * n;
  const double* B = a.B + (size_t)cls * n * dm.KIN;
  double* LT = a.LT + (size_t)cls * dm.KIN * n;
  for (int idx = threadIdx.x; idx < dm.KIN * n; idx += blockDim.x) {
    const int k = idx / n, r = idx % n;
    double s = 0.0;
    for (int j = 0; j < n; ++j) s = fma(Ai[(size_t)r * n + j], B[(size_t)j * dm.KIN + k], s);
    LT[idx] = s;
  }
  if (a.PT && a.R && dm.nr > 0) {
    const double* R = a.R + (size_t)cls * n * dm.nr;
    double* PT = a.PT + (size_t)cls * dm.nr * n;
    for (int idx = threadIdx.x; idx < dm.nr * n; idx += blockDim.x) {
      const int k = idx / n, r = idx % n;
      double s = 0.0;
      for (int j = 0; j < n; ++j) s = fma(Ai[(size_t)r * n + j], R[(size_t)j * dm.nr + k], s);
      PT[idx] = s;
    }
  }
  if (a.AinvT) {
    double* AT = a.AinvT + (size_t)cls * n * n;
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
      const int j = idx / n, r = idx % n;
      AT[idx] = Ai[(size_t)r * n + j];
    }
  }
}

// ---------------------------------------------------------------------------
// Analytic fields at element tensor points (nodal interpolation = project,
// SPEC.md:117-121; forcing at Gauss points for (f,v)_K).
// ---------------------------------------------------------------------------
__global__ void k_eval_field(const ihdg_field_args a) {
  Geo geo;
  geo.init(a.g, 1);
  const int D = geo.D;
  int npts = 1;
  for (int ax = 0; ax < D; ++ax) npts *= a.npts1d;
  const int64_t total = geo.nloc * npts;
  double* out0 = a.out + (a.out_ghost ? geo.ls * a.out_stride : 0) + a.out_offset;
  const int np = 2 + D;
  for (int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gid < total;
       gid += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = gid / npts;
    int pt = (int)(gid % npts);
    int64_t idx[3];
    geo.multi_index(e, idx);
    double x[3];
    for (int ax = 0; ax < D; ++ax) {
      const int ia = pt % a.npts1d;
      pt /= a.npts1d;
      // same rounding as mesh.py element_points: (lo + i h) + (0.5 h) (ref + 1)
      const double orig = __dadd_rn(a.lo[ax], __dmul_rn((double)idx[ax], a.h[ax]));
      x[ax] = __dadd_rn(orig, __dmul_rn(__dmul_rn(0.5, a.h[ax]), __dadd_rn(a.ref1d[ia], 1.0)));
    }
    double v = 0.0;
    for (int m = 0; m < a.nmodes; ++m) {
      const double* P = a.params + m * np;
      if (a.kind == 0) {
        double arg = P[1 + D];
        for (int ax = 0; ax < D; ++ax) arg = fma(2.0 * M_PI * P[1 + ax], x[ax], arg);
        v += P[0] * sin(arg);
      } else {
        double r2 = 0.0;
        for (int ax = 0; ax < D; ++ax) {
          const double dx = x[ax] - P[1 + ax];
          r2 = fma(dx, dx, r2);
        }
        const double w = P[1 + D];
        v += P[0] * exp(-r2 / (2.0 * w * w));
      }
    }
    out0[e * a.out_stride + (gid % npts)] = v;
  }
}

// b[e][i] = jac * sum_q prod_a Bq[i_a][q_a] fq[e][q]
__global__ void k_quad_project(const ihdg_quad_args a) {
  Geo geo;
  geo.init(a.g, 1);
  const int D = geo.D;
  const int N1 = a.g.order + 1;
  int NP = 1, NQ = 1;
  for (int ax = 0; ax < D; ++ax) {
    NP *= N1;
    NQ *= a.nq;
  }
  const int64_t total = geo.nloc * NP;
  for (int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gid < total;
       gid += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = gid / NP;
    const int i = (int)(gid % NP);
    int ia[3] = {0, 0, 0};
    int ii = i;
    for (int ax = 0; ax < D; ++ax) {
      ia[ax] = ii % N1;
      ii /= N1;
    }
    const double* f = a.fq + e * NQ;
    double s = 0.0;
    for (int q = 0; q < NQ; ++q) {
      int qq = q;
      double w = 1.0;
      for (int ax = 0; ax < D; ++ax) {
        w *= a.Bq[ia[ax] * a.nq + qq % a.nq];
        qq /= a.nq;
      }
      s = fma(w, f[q], s);
    }
    a.out[e * a.out_stride + a.out_offset + i] = a.jac * s;
  }
}

// ---------------------------------------------------------------------------
// Single-valued trace on every face in mesh.py order (mesh.py:89-125).
// ---------------------------------------------------------------------------
__global__ void k_extract_trace(const ihdg_trace_args a) {
  Geo geo;
  geo.init(a.g, 1);
  const int D = geo.D;
  const int N1 = a.g.order + 1;
  const int M = a.g.ncomp;
  int NP = 1, NF = 1;
  for (int ax = 0; ax < D; ++ax) NP *= N1;
  for (int ax = 0; ax < D - 1; ++ax) NF *= N1;
  const int NV = M * NP;
  // faces per axis
  int64_t off[4] = {0, 0, 0, 0};
  int64_t ntan[3], planes[3];
  for (int ax = 0; ax < D; ++ax) {
    ntan[ax] = 1;
    for (int b = 0; b < D; ++b)
      if (b != ax) ntan[ax] *= geo.c[b];
    planes[ax] = geo.c[ax] + (geo.per[ax] ? 0 : 1);
    off[ax + 1] = off[ax] + planes[ax] * ntan[ax];
  }
  const int64_t nfaces = off[D];
  const double* u0 = a.u + geo.ls * NV;
  for (int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gid < nfaces * NF;
       gid += (int64_t)gridDim.x * blockDim.x) {
    const int64_t fid = gid / NF;
    const int n = (int)(gid % NF);
    int ax = 0;
    while (fid >= off[ax + 1]) ++ax;
    const int64_t lf = fid - off[ax];
    const int64_t plane = lf / ntan[ax];
    int64_t tl = lf % ntan[ax];
    int64_t idx[3] = {0, 0, 0};
    for (int b = 0; b < D; ++b) {
      if (b == ax) continue;
      idx[b] = tl % geo.c[b];
      tl /= geo.c[b];
    }
    auto elem = [&](int64_t ia) {
      int64_t e = 0;
      for (int b = 0; b < D; ++b) e += (b == ax ? ia : idx[b]) * geo.stride[b];
      return e;
    };
    const int f_hi = 2 * ax + 1, f_lo = 2 * ax;
    double v = 0.0;
    if (plane > 0 && plane < geo.c[ax]) {
      const int64_t eo = elem(plane - 1), en = elem(plane);
      const int vo = face_node_vidx(D, N1, f_hi, n), vn = face_node_vidx(D, N1, f_lo, n);
      for (int c = 0; c < M; ++c)
        v += a.w_int_own[ax][c] * u0[eo * NV + c * NP + vo] + a.w_int_nbr[ax][c] * u0[en * NV + c * NP + vn];
    } else if (plane == 0 && geo.per[ax]) {
      const int64_t eo = elem(geo.c[ax] - 1), en = elem(0);
      const int vo = face_node_vidx(D, N1, f_hi, n), vn = face_node_vidx(D, N1, f_lo, n);
      for (int c = 0; c < M; ++c)
        v += a.w_int_own[ax][c] * u0[eo * NV + c * NP + vo] + a.w_int_nbr[ax][c] * u0[en * NV + c * NP + vn];
    } else if (plane == 0) {
      const int64_t eo = elem(0);
      const int vo = face_node_vidx(D, N1, f_lo, n);
      for (int c = 0; c < M; ++c) v += a.w_lo[ax][c] * u0[eo * NV + c * NP + vo];
    } else {
      const int64_t eo = elem(geo.c[ax] - 1);
      const int vo = face_node_vidx(D, N1, f_hi, n);
      for (int c = 0; c < M; ++c) v += a.w_hi[ax][c] * u0[eo * NV + c * NP + vo];
    }
    a.trace[gid] = v;
  }
}

__global__ void k_finalize(const ihdg_finalize_args a) {
  if (a.state->status != IHDG_RUNNING) return;  // later sweeps are no-ops
  const int64_t rl = a.row_len > 0 ? a.row_len : 1;
  finalize_block(a.tile_partials, a.n_tiles / rl, rl, a.state, a.norm_hist);
}

// Fixed-order sum of n partials (256 virtual lanes, then a fixed tree), the
// same order as finalize_block.  Every thread of the CTA must call it.
__device__ inline double fixed_sum(const double* parts, int64_t n) {
  __shared__ double red[256];
  __syncthreads();
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    double s = 0.0;
    for (int64_t i = v; i < n; i += 256) s += __ldcg(parts + i);
    red[v] = s;
  }
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    for (int v = threadIdx.x; v < w; v += blockDim.x) red[v] += red[v + w];
    __syncthreads();
  }
  return red[0];
}

constexpr int ERR_TE = 8;   // elements per error tile

// K5: ||u - u^e||^2 per tile by Gauss quadrature, then
// (mode 1) the exact-solution stopping rule in the last CTA.
__global__ void k_error_norm(const ihdg_error_args a) {
  ihdg_iter_state* st = a.state;
  if (a.mode != 0 && st->status != IHDG_RUNNING) return;   // later sweeps are no-ops
  __shared__ double vq_s[16 * 8];
  __shared__ double wq_s[16];
  __shared__ double red[256];
  __shared__ int last_s;
  const int d = a.g.dim, n1 = a.g.order + 1, m = a.g.ncomp, nq = a.nq;
  for (int i = threadIdx.x; i < nq * n1; i += blockDim.x) vq_s[i] = a.vq[i];
  for (int i = threadIdx.x; i < nq; i += blockDim.x) wq_s[i] = a.wq[i];
  int np = 1, nqd = 1;
  for (int i = 0; i < d; ++i) {
    np *= n1;
    nqd *= nq;
  }
  const int nv = m * np;
  Geo geo;
  geo.init(a.g, ERR_TE);
  const double* u = a.u + geo.ls * nv;
  __syncthreads();
  for (int64_t tile = blockIdx.x; tile < geo.ntiles; tile += gridDim.x) {
    int64_t e0;
    int nt;
    geo.tile_range(tile, ERR_TE, e0, nt);
    double acc = 0.0;
    const int items = nt * m * nqd;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
      const int t = it / (m * nqd), rem = it - t * m * nqd, c = rem / nqd, q = rem - c * nqd;
      int qa[3] = {q % nq, (q / nq) % nq, q / (nq * nq)};
      const double* ue = u + (e0 + t) * nv + c * np;
      double v = 0.0;
      for (int n = 0; n < np; ++n) {
        double w = vq_s[qa[0] * n1 + n % n1];
        if (d > 1) w *= vq_s[qa[1] * n1 + (n / n1) % n1];
        if (d > 2) w *= vq_s[qa[2] * n1 + n / (n1 * n1)];
        v = fma(w, ue[n], v);
      }
      double wt = wq_s[qa[0]];
      if (d > 1) wt *= wq_s[qa[1]];
      if (d > 2) wt *= wq_s[qa[2]];
      const double diff = v - a.ue_q[((e0 + t) * m + c) * (int64_t)nqd + q];
      acc = fma(a.comp_w[c] * wt * diff, diff, acc);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) a.err_partials[tile] = a.jac * red[0];
    __syncthreads();
  }
  // last CTA: reduce (mode 0: initial error; mode 1: stop rule)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned tk = atomicAdd(&st->ticket, 1u);
    last_s = (tk == gridDim.x - 1);
  }
  __syncthreads();
  if (!last_s) return;
  __threadfence();
  const double err = sqrt(fixed_sum(a.err_partials, geo.ntiles));
  if (a.mode == 0) {
    if (threadIdx.x == 0) {
      st->last_err = err;
      st->ticket = 0u;
      __threadfence();
    }
    return;
  }
  // the sweep's tile partials, in the rows of finalize_block
  const int64_t srows = geo.D == 1 ? 1 : geo.nlay;
  const double norm = sqrt(rows_sum(a.succ_partials, srows, a.n_succ / srows));
  if (threadIdx.x == 0) {
    const int it = st->iters + 1;
    st->iters = it;
    if (a.norm_hist != nullptr && it <= st->max_iters) a.norm_hist[it - 1] = norm;
    if (a.err_hist != nullptr && it <= st->max_iters) a.err_hist[it - 1] = err;
    if (it == 1) st->first_norm = norm;
    st->last_norm = norm;
    int status = IHDG_RUNNING;
    if (!(norm == norm) || !(err == err)) status = IHDG_NAN;
    else if (a.mode == 2 ? (err < st->tol) : (fabs(err - st->last_err) < st->tol)) status = IHDG_CONVERGED;
    else if (it > 1 && norm > st->diverge_factor * st->first_norm) status = IHDG_DIVERGED;
    else if (it >= st->max_iters) status = IHDG_MAXITER;
    st->last_err = err;
    st->status = status;
    st->ticket = 0u;
    __threadfence();
  }
}


// ---------------------------------------------------------------------------
// K6: per-iteration diagnostics of iteration.run (SPEC.md:320-323, 341-349,
// 398).  Diagnostic mode only (the reference computes them single-threaded
// after the barrier); not on the sweep path.
// ---------------------------------------------------------------------------

// err2[e] = J sum_c comp_w[c] |(C^T x .. x C^T)(u - r)_{e,c}|^2, one element
// per CTA pass: the difference is staged in shared memory and one exact
// triangular pass per axis runs over the node lines (same factorisation as
// the sweep's stopping norm, M1 = C C^T).
__global__ void k_elem_error(const ihdg_elem_error_args a) {
  __shared__ double x_s[IHDG_MAX_COMP * 512];
  __shared__ double c_s[64];
  __shared__ double red[128];
  const int d = a.g.dim, n1 = a.g.order + 1, m = a.g.ncomp;
  int np = 1;
  for (int i = 0; i < d; ++i) np *= n1;
  const int nv = m * np, lpl = np / n1;
  for (int i = threadIdx.x; i < n1 * n1; i += blockDim.x) c_s[i] = a.chol1d[i];
  Geo geo;
  geo.init(a.g, 1);
  const double* u = a.u + geo.ls * nv;
  const double* r = a.r + geo.ls * nv;
  __syncthreads();
  for (int64_t e = blockIdx.x; e < geo.nloc; e += gridDim.x) {
    for (int i = threadIdx.x; i < nv; i += blockDim.x) x_s[i] = u[e * nv + i] - r[e * nv + i];
    __syncthreads();
    double acc = 0.0;
    int mul = 1;
    for (int ax = 0; ax < d; ++ax) {
      const bool last_ax = ax == d - 1;
      for (int ln = threadIdx.x; ln < m * lpl; ln += blockDim.x) {
        const int c = ln / lpl;
        int rem = ln - c * lpl, base = c * np, mb = 1;
        for (int b = 0; b < d; ++b) {
          if (b != ax) {
            base += (rem % n1) * mb;
            rem /= n1;
          }
          mb *= n1;
        }
        double xv[8];
        for (int i = 0; i < n1; ++i) xv[i] = x_s[base + i * mul];
        for (int i = 0; i < n1; ++i) {
          double y = 0.0;
          for (int ip = i; ip < n1; ++ip) y = fma(c_s[ip * n1 + i], xv[ip], y);
          if (last_ax) acc = fma(a.comp_w[c] * y, y, acc);
          else x_s[base + i * mul] = y;
        }
      }
      __syncthreads();
      mul *= n1;
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 64; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const double e2 = a.jac * red[0];
      a.err2[e] = e2;
      if (a.flags != nullptr) a.flags[e] = (uint8_t)(e2 < a.tol * a.tol ? 1 : 0);
    }
    __syncthreads();
  }
}

// e2[f] = Jf_axis |(C^T x .. x C^T) t_f|^2 for every face of t (mesh.py face
// order, as written by k_extract_trace)
__global__ void k_face_energy(const ihdg_face_energy_args a) {
  Geo geo;
  geo.init(a.g, 1);
  const int D = geo.D, n1 = a.g.order + 1;
  int nf = 1;
  for (int i = 0; i < D - 1; ++i) nf *= n1;
  int64_t off[4] = {0, 0, 0, 0};
  for (int ax = 0; ax < D; ++ax) {
    int64_t ntan = 1;
    for (int b = 0; b < D; ++b)
      if (b != ax) ntan *= geo.c[b];
    off[ax + 1] = off[ax] + (geo.c[ax] + (geo.per[ax] ? 0 : 1)) * ntan;
  }
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < off[D];
       f += (int64_t)gridDim.x * blockDim.x) {
    int ax = 0;
    while (f >= off[ax + 1]) ++ax;
    double x[64];
    for (int i = 0; i < nf; ++i) x[i] = a.t[f * nf + i] - (a.t_ref != nullptr ? a.t_ref[f * nf + i] : 0.0);
    // tangential passes: axis 0 of the face (fastest), then axis 1
    double acc = 0.0;
    if (D == 1) {
      acc = x[0] * x[0];
    } else {
      const int nt = D - 1;
      int mul = 1;
      for (int b = 0; b < nt; ++b) {
        const bool last_b = b == nt - 1;
        for (int ln = 0; ln < nf / n1; ++ln) {
          const int base = (b == 0) ? ln * n1 : ln;
          for (int i = 0; i < n1; ++i) {
            double y = 0.0;
            for (int ip = i; ip < n1; ++ip) y = fma(a.chol1d[ip * n1 + i], x[base + ip * mul], y);
            if (last_b) acc = fma(y, y, acc);
            else x[base + i * mul] = y;  // in place: later rows read only ip >= i' > i
          }
        }
        mul *= n1;
      }
    }
    a.e2[f] = a.jac_face[ax] * acc;
  }
}

// *out = fixed-order sum of n values (one CTA)
__global__ void k_fixed_total(const double* v, int64_t n, double* out) {
  const double s = fixed_sum(v, n);
  if (threadIdx.x == 0) *out = s;
}

// out[r] = sum of row r of the tile partials (warp_row_sum, the inner sums
// of rows_sum): one warp per row
__global__ void k_layer_sums(const double* parts, int64_t n_rows, int64_t row_len, double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n_rows; r += nw) {
    const double s = warp_row_sum(parts + r * row_len, row_len, lane);
    if (lane == 0) out[r] = s;
  }
}

// Halo pack / unpack: element-local DOF entries idx[0..n_idx) of every
// element of one layer, between the ghost-padded state and a packed
// [layer elems][n_idx] buffer.  layer: 0 = ghost_lo, 1 = first local,
// 2 = last local, 3 = ghost_hi (rows of the padded buffer).
__global__ void k_halo_copy(const ihdg_halo_args a, int unpack) {
  Geo geo;
  geo.init(a.g, 1);
  const int64_t ls = geo.ls;
  const int64_t nv = (int64_t)a.g.ncomp * ipow(a.g.order + 1, a.g.dim);
  const int64_t row = a.layer == 0 ? 0 : (a.layer == 1 ? 1 : (a.layer == 2 ? geo.nlay : geo.nlay + 1));
  double* base = a.buf + row * ls * nv;
  const int64_t total = ls * a.n_idx;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / a.n_idx;
    const int j = (int)(t - e * a.n_idx);
    double* p = base + e * nv + a.idx[j];
    if (unpack) *p = a.packed[t];
    else a.packed[t] = *p;
  }
}

}  // namespace ihdg
