// Streaming iHDG-II sweep for sm_100a (K2 + K3, production path).
//
// One persistent CTA per SM walks tiles of E consecutive elements of one
// element layer (a row segment).  The FieldState layout is element-major, so
// a tile of s and of u^k is one contiguous byte range:
//
//   producer warp : cp.async.bulk (TMA, 1D) of the s and u^k tiles into a
//                   NS-stage shared-memory ring, completion on an mbarrier
//                   (complete_tx), plus 8-byte cp.async gathers of the
//                   neighbour face nodes that are not inside the tile
//                   (other layers, tile ends) -> per-stage halo buffer.
//   consumer warps: q = neighbour face scalars (TraceSnapshot)
//                   from the tile / halo; u^{k+1} = s + L q with the class
//                   operator L = A^-1 B (lifted apply_local)
//                   held in REGISTERS (thread = row of L, loaded once per
//                   kernel); u^{k+1} staged in shared memory and written back
//                   with one cp.async.bulk store per tile; delta = u^{k+1}-u^k
//                   -> mass-weighted norm by sum-factorised Cholesky passes.
//
// HBM traffic per element-DOF: read s, read u^k, write u^{k+1} = 24 B
// (SURVEY.md 8d); neighbour face reads hit L2 because concurrently processed
// tiles are spatially adjacent (row-major tile order).
#pragma once

#include "ihdg_common.cuh"
#include "ihdg_kernels.cuh"

namespace ihdg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_bar(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

// D dims, N1 = p+1, M comps, NCF coupled faces, NWC weighted comps per face,
// E elements per tile, NS pipeline stages, G consumer groups (split E).
template <int D, int N1, int M, int NCF, int NWC, int E, int NS, int G>
struct SCfg {
  static constexpr int NP = Pow<N1, D>::v;
  static constexpr int NV = M * NP;
  static constexpr int NF = Pow<N1, D - 1>::v;
  static constexpr int NFACE = 2 * D;
  static constexpr int KC = NCF * NF;            // compacted neighbour scalars
  static constexpr int RP = round_up(NV, 32);    // row threads per group
  static constexpr int NC = G * RP;              // consumer threads
  static constexpr int NCW = NC / 32;
  static constexpr int NT = NC + 32;             // + producer warp
  static constexpr int EG = E / G;               // elements per group
  static constexpr int TILE = E * NV;            // doubles
  static constexpr int HALO = E * NCF * NWC * NF;
  static constexpr int STAGE = 2 * TILE + HALO;
  // shared memory carve (doubles)
  static constexpr int OFF_STAGE = 0;
  static constexpr int OFF_OUT = NS * STAGE;
  static constexpr int OFF_D = OFF_OUT + 2 * TILE;
  static constexpr int OFF_T = OFF_D + TILE;
  static constexpr int OFF_Q = OFF_T + TILE;
  static constexpr int OFF_PART = OFF_Q + E * KC;
  static constexpr int OFF_CHOL = OFF_PART + E;
  static constexpr int N_DBL = OFF_CHOL + N1 * N1;
  static constexpr size_t BYTES = (size_t)N_DBL * sizeof(double) + 2 * NS * sizeof(uint64_t);
  static_assert(EG % 4 == 0, "elements per group must be a multiple of 4");
  static_assert(KC % 2 == 0, "compacted neighbour count must be even");
  static_assert((TILE * sizeof(double)) % 16 == 0, "tile bytes must be 16-byte multiples");
};

template <int D, int N1, int M, int NCF, int NWC, int E, int NS, int G>
__global__ void __launch_bounds__(SCfg<D, N1, M, NCF, NWC, E, NS, G>::NT, 1)
    k_sweep_stream(const ihdg_sweep_args a) {
  using C = SCfg<D, N1, M, NCF, NWC, E, NS, G>;
  constexpr int NP = C::NP, NV = C::NV, NF = C::NF, NFACE = C::NFACE, KC = C::KC;
  constexpr int RP = C::RP, NC = C::NC, NCW = C::NCW, EG = C::EG, TILE = C::TILE;

  extern __shared__ __align__(128) double sm[];
  double* out_s = sm + C::OFF_OUT;
  double* d_s = sm + C::OFF_D;
  double* t_s = sm + C::OFF_T;
  double* q_s = sm + C::OFF_Q;
  double* part_s = sm + C::OFF_PART;
  double* c_s = sm + C::OFF_CHOL;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sm + C::N_DBL);
  uint64_t* empty_bar = full_bar + NS;

  __shared__ int fv_s[NFACE][NF];
  __shared__ int cf_s[NCF];                 // coupled local faces
  __shared__ int wc_s[NCF][NWC];            // weighted components
  __shared__ double ww_s[NCF][NWC];         // their weights
  __shared__ int mask_s[E];                 // missing-neighbour bits
  __shared__ int cls_s[E];
  __shared__ int fast_s;
  __shared__ int last_s;

  ihdg_iter_state* st = a.state;
  if (st->status != IHDG_RUNNING) return;

  const int tid = threadIdx.x;
  Geo geo;
  geo.init(a.g, E);
  const int64_t ls = geo.ls;
  const double* __restrict__ uo = a.u_old + ls * NV;
  double* __restrict__ un = a.u_new + ls * NV;

  for (int i = tid; i < NFACE * NF; i += blockDim.x) fv_s[i / NF][i % NF] = face_node_vidx(D, N1, i / NF, i % NF);
  for (int i = tid; i < N1 * N1; i += blockDim.x) c_s[i] = a.chol1d[i];
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
      mbar_init(&full_bar[s], 1 + 32);
      mbar_init(&empty_bar[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int fast_class = a.class_of_mask[0];
  const int64_t ntiles = geo.ntiles;
  const uint32_t tile_bytes = (uint32_t)(TILE * sizeof(double));

  if (tid >= NC) {
    // ============================ producer warp ============================
    const int lane = tid - NC;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int stage = it % NS;
      if (it >= NS) mbar_wait(&empty_bar[stage], ((it / NS) - 1) & 1);
      double* sst = sm + stage * C::STAGE;
      double* ust = sst + TILE;
      double* hst = ust + TILE;
      TileInfo ti;
      ti.init(geo, tile, E);
      const int64_t e0 = ti.e0;
      const int nt = ti.nt;
      if (lane == 0) {
        const uint32_t bytes = (uint32_t)(nt * NV * sizeof(double));
        mbar_arrive_expect_tx(&full_bar[stage], 2 * bytes);
        bulk_g2s(sst, a.s + e0 * NV, bytes, &full_bar[stage]);
        bulk_g2s(ust, uo + e0 * NV, bytes, &full_bar[stage]);
      }
      // neighbour face nodes that are not inside this tile
      for (int p = lane; p < nt * NCF; p += 32) {
        const int t = p / NCF, ci = p % NCF;
        const int f = cf_s[ci];
        const bool axis0 = (f >> 1) == 0;
        if (axis0 && !((f == 0 && t == 0) || (f == 1 && t == nt - 1))) continue;
        if (ti.mask(t, D) & (1 << f)) continue;
        const double* src = uo + ti.nbr(t, f) * NV;
        double* dst = hst + ((t * NCF + ci) * NWC) * NF;
#pragma unroll
        for (int j = 0; j < NWC; ++j) {
          const double* sc = src + wc_s[ci][j] * NP;
#pragma unroll
          for (int n = 0; n < NF; ++n) cp_async8(dst + j * NF + n, sc + fv_s[f ^ 1][n]);
        }
      }
      cp_async_arrive_noinc(&full_bar[stage]);
    }
  } else {
    // ============================ consumer warps ===========================
    const int r = tid % RP;
    const int g = tid / RP;
    const bool rv = r < NV;
    const int warp = tid >> 5, lane = tid & 31;
    // lifted operator of the interior class, one row per thread, in registers
    double Lr[KC];
#pragma unroll
    for (int k = 0; k < KC; ++k) {
      const int col = cf_s[k / NF] * NF + (k % NF);
      Lr[k] = rv ? __ldg(a.LT + ((size_t)fast_class * (NFACE * NF) + col) * NV + r) : 0.0;
    }
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int stage = it % NS;
      const int ob = it & 1;
      TileInfo ti;
      ti.init(geo, tile, E);
      const int64_t e0 = ti.e0;
      const int nt = ti.nt;
      if (tid < E) {
        int mask = 0, cls = -1;
        if (tid < nt) {
          mask = ti.mask(tid, D);
          cls = a.class_of_mask[mask];
        }
        mask_s[tid] = mask;
        cls_s[tid] = cls;
      }
      mbar_wait(&full_bar[stage], (it / NS) & 1);
      if (tid == 0 && it >= 2) bulk_wait_read<1>();
      consumer_bar(NC);
      if (tid == 0) {
        int fast = 1;
        for (int t = 0; t < nt; ++t) fast &= (cls_s[t] == fast_class);
        fast_s = fast;
      }
      const double* sst = sm + stage * C::STAGE;
      const double* ust = sst + TILE;
      const double* hst = ust + TILE;
      // ---- neighbour face scalars q[t][k] --------------------------------
      for (int idx = tid; idx < E * KC; idx += NC) {
        const int t = idx / KC, k = idx % KC;
        const int ci = k / NF, n = k % NF;
        const int f = cf_s[ci];
        double v = 0.0;
        if (t < nt && !(mask_s[t] & (1 << f))) {
          const bool axis0 = (f >> 1) == 0;
          const bool in_tile = axis0 && !((f == 0 && t == 0) || (f == 1 && t == nt - 1));
          if (in_tile) {
            const double* src = ust + (t + (f == 0 ? -1 : 1)) * NV + fv_s[f ^ 1][n];
#pragma unroll
            for (int j = 0; j < NWC; ++j) v = fma(ww_s[ci][j], src[wc_s[ci][j] * NP], v);
          } else {
            const double* src = hst + ((t * NCF + ci) * NWC) * NF + n;
#pragma unroll
            for (int j = 0; j < NWC; ++j) v = fma(ww_s[ci][j], src[j * NF], v);
          }
        }
        q_s[idx] = v;
      }
      consumer_bar(NC);
      // ---- lifted local solve u^{k+1} = s + L q ---------------------------
      double* outb = out_s + ob * TILE;
      if (rv) {
        if (fast_s) {
#pragma unroll
          for (int tb = 0; tb < EG; tb += 4) {
            double acc[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int t = g * EG + tb + c;
              acc[c] = (t < nt) ? sst[t * NV + r] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < KC; k += 2) {
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const int t = g * EG + tb + c;
                const double2 qv = *reinterpret_cast<const double2*>(q_s + t * KC + k);
                acc[c] = fma(Lr[k], qv.x, acc[c]);
                acc[c] = fma(Lr[k + 1], qv.y, acc[c]);
              }
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int t = g * EG + tb + c;
              if (t < nt) {
                outb[t * NV + r] = acc[c];
                d_s[t * NV + r] = acc[c] - ust[t * NV + r];
              }
            }
          }
        } else {
          for (int tt = 0; tt < EG; ++tt) {
            const int t = g * EG + tt;
            if (t >= nt) continue;
            const double* __restrict__ Lc = a.LT + (size_t)cls_s[t] * (NFACE * NF) * NV + r;
            double acc = sst[t * NV + r];
            for (int k = 0; k < KC; ++k) {
              const int col = cf_s[k / NF] * NF + (k % NF);
              acc = fma(__ldg(Lc + (size_t)col * NV), q_s[t * KC + k], acc);
            }
            outb[t * NV + r] = acc;
            d_s[t * NV + r] = acc - ust[t * NV + r];
          }
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[stage]);
      consumer_bar(NC);
      if (tid == 0) {
        bulk_s2g(un + e0 * NV, outb, (uint32_t)(nt * NV * sizeof(double)));
        bulk_commit();
      }
      // ---- ||delta||_M^2 by sum-factorised Cholesky passes ----------------
      double* src = d_s;
      double* dst = t_s;
      int mul = 1;
#pragma unroll
      for (int ax = 0; ax < D; ++ax) {
        for (int i = tid; i < nt * NV; i += NC) {
          const int t = i / NV, rem = i % NV;
          const int n = rem % NP;
          const int ia = (n / mul) % N1;
          const int base = t * NV + rem - ia * mul;
          double v = 0.0;
#pragma unroll
          for (int ip = 0; ip < N1; ++ip)
            if (ip >= ia) v = fma(c_s[ip * N1 + ia], src[base + ip * mul], v);
          dst[i] = v;
        }
        consumer_bar(NC);
        double* tmp = src;
        src = dst;
        dst = tmp;
        mul *= N1;
      }
      for (int t = warp; t < nt; t += NCW) {
        double s = 0.0;
        for (int i = lane; i < NV; i += 32) {
          const double v = src[t * NV + i];
          s = fma(a.comp_w[i / NP] * v, v, s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) part_s[t] = a.jac * s;
      }
      consumer_bar(NC);
      if (tid == 0) {
        double s = 0.0;
        for (int t = 0; t < nt; ++t) s += part_s[t];
        a.tile_partials[tile] = s;
      }
    }
    if (tid == 0) bulk_wait<0>();
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
