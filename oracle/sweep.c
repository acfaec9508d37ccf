/*
 * CPU ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/ihdg_oracle.py header).
 *
 * C/OpenMP restatement of the reference's native element map
 * `ihdg._kernels._sweep_cy` (pkg/setup.py:13-19, compiled there with
 * -O3 -fopenmp; source absent from /root/reference).  One sweep of iHDG-II in
 * the reference's own algorithm: for every element, build
 * the RHS from the frozen iterate-k neighbour face data (TraceSnapshot,
 * SPEC.md:240-243) and solve with the factor-once dense LU,
 * element-disjoint writes into the k+1 buffer.  Also returns
 * sum_K sum_c delta_c^T M delta_c for the successive-difference stopping rule
 * (PAPER.md:1308-1311).
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

int32_t oracle_max_threads(void) { return (int32_t)omp_get_max_threads(); }

double oracle_sweep(int64_t nel, int32_t nv, int32_t nface, const int64_t* nbr, const int32_t* cls,
                    const double* LU, const int32_t* piv, int32_t nr, const int32_t* rows,
                    const int32_t* cols, const double* blk, const double* rhs, const double* u_old,
                    double* u_new, int32_t npn, const double* mass, int32_t m, int32_t nthreads) {
  if (nthreads > 0) omp_set_num_threads(nthreads);
  double total = 0.0;
#pragma omp parallel reduction(+ : total)
  {
    double* r = (double*)malloc(sizeof(double) * (size_t)nv);
    double* g = (double*)malloc(sizeof(double) * (size_t)nr);
    double* dl = (double*)malloc(sizeof(double) * (size_t)npn);
#pragma omp for schedule(static)
    for (int64_t e = 0; e < nel; ++e) {
      const int c = cls[e];
      const double* lu = LU + (size_t)c * nv * nv;
      const int32_t* pv = piv + (size_t)c * nv;
      memcpy(r, rhs + (size_t)e * nv, sizeof(double) * (size_t)nv);
      /* RHS builder: neighbour iterate-k face data */
      for (int f = 0; f < nface; ++f) {
        const int64_t nb = nbr[e * nface + f];
        if (nb < 0) continue;
        const double* un = u_old + (size_t)nb * nv;
        const int32_t* cf = cols + (size_t)f * nr;
        const int32_t* rf = rows + (size_t)f * nr;
        for (int j = 0; j < nr; ++j) g[j] = un[cf[j]];
        const double* B = blk + ((size_t)c * nface + f) * nr * nr;
        for (int i = 0; i < nr; ++i) {
          double s = 0.0;
          for (int j = 0; j < nr; ++j) s += B[(size_t)i * nr + j] * g[j];
          r[rf[i]] += s;
        }
      }
      /* LU solve (getrf layout: unit-lower L, U, sequential row interchanges) */
      for (int i = 0; i < nv; ++i) {
        const int p = pv[i];
        if (p != i) {
          const double t = r[i];
          r[i] = r[p];
          r[p] = t;
        }
      }
      for (int i = 1; i < nv; ++i) {
        double s = r[i];
        const double* li = lu + (size_t)i * nv;
        for (int j = 0; j < i; ++j) s -= li[j] * r[j];
        r[i] = s;
      }
      for (int i = nv - 1; i >= 0; --i) {
        double s = r[i];
        const double* ui = lu + (size_t)i * nv;
        for (int j = i + 1; j < nv; ++j) s -= ui[j] * r[j];
        r[i] = s / ui[i];
      }
      /* write + successive-difference mass norm */
      const double* uo = u_old + (size_t)e * nv;
      double* out = u_new + (size_t)e * nv;
      for (int cc = 0; cc < m; ++cc) {
        for (int i = 0; i < npn; ++i) dl[i] = r[cc * npn + i] - uo[cc * npn + i];
        for (int i = 0; i < npn; ++i) {
          double s = 0.0;
          const double* mi = mass + (size_t)i * npn;
          for (int j = 0; j < npn; ++j) s += mi[j] * dl[j];
          total += dl[i] * s;
        }
      }
      memcpy(out, r, sizeof(double) * (size_t)nv);
    }
    free(r);
    free(g);
    free(dl);
  }
  return total;
}
