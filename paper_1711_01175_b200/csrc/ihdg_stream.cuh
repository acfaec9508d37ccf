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

// Optional per-role cycle counters (profiling build, -DIHDG_WS_PROF; tools/ws_roles.py).
#ifdef IHDG_WS_PROF
__device__ unsigned long long g_ws_prof[16];
// per-CTA shared counters, flushed once per CTA (V3_FLUSH) to keep the
// measurement from perturbing the kernel
#define V3_DECL __shared__ unsigned long long prof_s[16]; if (threadIdx.x < 16) prof_s[threadIdx.x] = 0ull;
#define V3_T0(v) const long long v = clock64()
#define V3_ACC(slot, v)                                                                              \
  do {                                                                                               \
    if ((threadIdx.x & 31) == 0) atomicAdd(&prof_s[slot], (unsigned long long)(clock64() - (v)));    \
  } while (0)
#define V3_FLUSH                                                                                     \
  do {                                                                                               \
    __syncthreads();                                                                                 \
    if (threadIdx.x < 16) atomicAdd(&g_ws_prof[threadIdx.x], prof_s[threadIdx.x]);                   \
  } while (0)
#else
#define V3_DECL
#define V3_T0(v)
#define V3_ACC(slot, v)
#define V3_FLUSH
#endif

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
// L2 prefetch of a global range (bytes % 16 == 0): raises the bytes in flight
// per SM beyond what the shared-memory stage ring can hold
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
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
// named barrier over a subset of warps (id 1..15; 0 is __syncthreads)
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
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
// D(8x8) += A(8x4, row) * B(4x8, col), fp64 tensor core (SASS DMMA.8x8x4).
// lane l holds A[l>>2][l&3], B[l&3][l>>2], D[l>>2][2(l&3)], D[l>>2][2(l&3)+1].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void consumer_bar(int n) { asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory"); }

// 32-bit tile geometry for the streaming kernel (host guarantees local
// element and tile counts < 2^31 and cells[0] % E == 0).  Tile = E
// consecutive elements of one axis-0 row.  Neighbour offsets across faces of
// axes >= 1 are the same for every element of the tile.
// Exact unsigned division by a runtime-invariant divisor (round-up method:
// q = (mulhi(n, m) + n) >> s for every 32-bit n); init once per kernel.
struct FastDiv {
  uint32_t m, s;
  __device__ __forceinline__ void init(uint32_t d) {
    s = d <= 1 ? 0 : 32 - __clz(d - 1);
    m = (uint32_t)(((1ull << 32) * ((1ull << s) - d)) / d + 1ull);
  }
  __device__ __forceinline__ int div(int n) const {
    return (int)(((unsigned long long)__umulhi((uint32_t)n, m) + (uint32_t)n) >> s);
  }
};

template <int D>
struct STile {
  int e0, nt, i0;
  int has[2 * D];   // neighbour exists across face f (axis >= 1 entries only)
  int off[2 * D];   // neighbour element offset across face f (axis >= 1)

  __device__ __forceinline__ void init(const ihdg_geom& g, int tile, int E, int nlay, int ls) {
    const int c0 = (int)g.cells[0];
    const int segs0 = c0 / E;
    const int xrow = tile / segs0;
    init_row(g, tile, xrow, D == 3 ? xrow / (int)g.cells[1] : xrow, segs0, E, nlay, ls);
  }
  // the same with the two divisions done by precomputed FastDiv (segs0 = c0 / E, c1)
  __device__ __forceinline__ void init(const ihdg_geom& g, int tile, int E, int nlay, int ls, int segs0,
                                       const FastDiv& dsegs0, const FastDiv& dc1) {
    const int xrow = dsegs0.div(tile);
    init_row(g, tile, xrow, D == 3 ? dc1.div(xrow) : xrow, segs0, E, nlay, ls);
  }
  __device__ __forceinline__ void init_row(const ihdg_geom& g, int tile, int xrow, int lay3, int segs0, int E, int nlay,
                                           int ls) {
    const int c0 = (int)g.cells[0];
    i0 = (tile - xrow * segs0) * E;
    e0 = xrow * c0 + i0;
    nt = E;
    int lay = xrow;      // local layer (D == 2)
    if (D == 3) {
      const int c1 = (int)g.cells[1];
      lay = lay3;
      const int i1 = xrow - lay * c1;
      // axis 1 (inside the layer)
      has[2] = (i1 > 0) || g.periodic[1];
      off[2] = i1 > 0 ? -c0 : (c1 - 1) * c0;
      has[3] = (i1 < c1 - 1) || g.periodic[1];
      off[3] = i1 < c1 - 1 ? c0 : -(c1 - 1) * c0;
    }
    if (D >= 2) {
      // layer axis (D-1): global index, ghost layers beyond the strip
      const int L = (int)g.cells[D - 1];
      const int jg = (int)g.layer_begin + lay;
      const int flo = 2 * (D - 1), fhi = flo + 1;
      int jl = jg - 1, jh = jg + 1;
      has[flo] = (jl >= 0) || g.periodic[D - 1];
      has[fhi] = (jh < L) || g.periodic[D - 1];
      if (jl < 0) jl = L - 1;
      if (jh >= L) jh = 0;
      int ll = jl - (int)g.layer_begin, lh = jh - (int)g.layer_begin;
      if (!(ll >= 0 && ll < nlay)) ll = -1;
      if (!(lh >= 0 && lh < nlay)) lh = nlay;
      off[flo] = (ll - lay) * ls;
      off[fhi] = (lh - lay) * ls;
    }
    has[0] = has[1] = 1;
    off[0] = -1;
    off[1] = 1;
  }
  __device__ __forceinline__ int face_has(int f) const {
    int v = 0;
#pragma unroll
    for (int k = 2; k < 2 * D; ++k) v = (f == k) ? has[k] : v;
    return v;
  }
  __device__ __forceinline__ int face_off(int f) const {
    int v = 0;
#pragma unroll
    for (int k = 2; k < 2 * D; ++k) v = (f == k) ? off[k] : v;
    return v;
  }
  // missing-neighbour mask of tile element t
  __device__ __forceinline__ int mask(int t, int c0, int per0) const {
    int m = 0;
    const int i = i0 + t;
    if (!per0) {
      if (i == 0) m |= 1;
      if (i == c0 - 1) m |= 2;
    }
#pragma unroll
    for (int f = 2; f < 2 * D; ++f)
      if (!has[f]) m |= 1 << f;
    return m;
  }
};

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
  static constexpr int EG = E / G;               // elements per group (DFMA norm)
  static constexpr int NRT = (NV + 7) / 8;       // DMMA row tiles
  static constexpr int KS = KC / 4;              // DMMA k steps
  static constexpr int NEG = E / 8;              // DMMA element groups
  static constexpr int RTW = (NRT + NCW - 1) / NCW;  // row tiles per consumer warp
  // 2D with p+1 <= 8: norm on the tensor core, software-pipelined one tile behind
  static constexpr bool PIPE = (D == 2 && N1 <= 8);
  static constexpr int UPW = (E * M + NCW - 1) / NCW;  // norm units per warp
  static constexpr int TILE = E * NV;            // doubles
  static constexpr int HALO = E * NCF * NWC * NF;
  static constexpr int STAGE = 2 * TILE + HALO;
  // shared memory carve (doubles)
  static constexpr int OFF_OUT = NS * STAGE;
  static constexpr int OFF_D = OFF_OUT + 2 * TILE;   // delta (PIPE: double buffer)
  static constexpr int OFF_T = OFF_D + TILE;         // DFMA pass scratch / delta buffer 1
  static constexpr int OFF_Q = OFF_T + TILE;
  static constexpr int OFF_RED = OFF_Q + E * KC;
  static constexpr int N_DBL = OFF_RED + 64;
  static constexpr size_t BYTES = (size_t)N_DBL * sizeof(double) + 2 * NS * sizeof(uint64_t);
  static_assert(EG % 4 == 0, "elements per group must be a multiple of 4");
  static_assert(KC % 4 == 0, "compacted neighbour count must be a multiple of 4 (DMMA k)");
  static_assert(E % 8 == 0, "tile must be a multiple of 8 elements (DMMA n)");
  static_assert(E <= 32, "one producer lane per tile element");
  static_assert(NCW <= 32, "warp partials fit one reduction row");
  static_assert((TILE * sizeof(double)) % 16 == 0, "tile bytes must be 16-byte multiples");
};

// ||Y||_F^2 of Y = C^T Delta C for the UPW (element, component) units of this
// warp (2D, tensor core).  Delta[j][i] = delta at node (i, j), zero padded to
// 8x8; cfr = C fragments.  Invalid units read zeros (uniform control flow).
template <int N1, int M, int NP, int NV, int E, int NCW, int UPW, int PS = 0>
__device__ __forceinline__ double norm_units_2d(const double* __restrict__ dbuf, int warp, int lane,
                                                const double (&cfr)[2], const double* comp_w) {
  double acc = 0.0;
  double r0[UPW], r1[UPW];
#pragma unroll
  for (int m = 0; m < UPW; ++m) {
    const int u = warp + m * NCW;
    const bool valid = u < E * M;
    const int uu = valid ? u : 0;
    const int t = uu / M, c = uu - (uu / M) * M;
    // element offset: plain (t NV) or padded element pairs (pair stride PS)
    const double* base = dbuf + (PS ? (t >> 1) * PS + (t & 1) * NV : t * NV) + c * NP;
    r0[m] = 0.0;
    r1[m] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int kk = 4 * ks + (lane & 3), nn = lane >> 2;
      const double b = (valid && kk < N1 && nn < N1) ? base[kk * N1 + nn] : 0.0;
      dmma_8x8x4(r0[m], r1[m], cfr[ks], b);   // R = C^T Delta
    }
  }
#pragma unroll
  for (int m = 0; m < UPW; ++m) {
    const int u = warp + m * NCW;
    const int c = (u < E * M ? u : 0) % M;
    double y0 = 0.0, y1 = 0.0;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int col = 4 * ks + (lane & 3);     // A fragment R[lane>>2][col]
      const int src = (lane & ~3) | (col >> 1);
      const double x0 = __shfl_sync(0xffffffffu, r0[m], src);
      const double x1 = __shfl_sync(0xffffffffu, r1[m], src);
      dmma_8x8x4(y0, y1, (col & 1) ? x1 : x0, cfr[ks]);  // Y = R C
    }
    const double w = comp_w[c];
    acc = fma(w * y0, y0, acc);
    acc = fma(w * y1, y1, acc);
  }
  return acc;
}

template <int D, int N1, int M, int NCF, int NWC, int E, int NS, int G>
__global__ void __launch_bounds__(SCfg<D, N1, M, NCF, NWC, E, NS, G>::NT, 1)
    k_sweep_stream(const ihdg_sweep_args a) {
  using C = SCfg<D, N1, M, NCF, NWC, E, NS, G>;
  constexpr int NP = C::NP, NV = C::NV, NF = C::NF, NFACE = C::NFACE, KC = C::KC;
  constexpr int RP = C::RP, NC = C::NC, NCW = C::NCW, EG = C::EG, TILE = C::TILE;
  constexpr int NRT = C::NRT, KS = C::KS, NEG = C::NEG, RTW = C::RTW, UPW = C::UPW;

  extern __shared__ __align__(16) double sm[];
  double* out_s = sm + C::OFF_OUT;
  double* d_s = sm + C::OFF_D;
  double* t_s = sm + C::OFF_T;
  double* q_s = sm + C::OFF_Q;
  double* red_s = sm + C::OFF_RED;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sm + C::N_DBL);
  uint64_t* empty_bar = full_bar + NS;

  __shared__ int fv_s[NFACE][NF];
  __shared__ int cf_s[NCF];                 // coupled local faces
  __shared__ int wc_s[NCF][NWC];            // weighted components
  __shared__ double ww_s[NCF][NWC];         // their weights
  __shared__ double chol_s[N1 * N1];
  __shared__ double cshift_s[N1 * N1];      // cshift[ia][k] = C[ia+k][ia] (0 past the end)
  __shared__ int qf_s[KC];                  // face of neighbour scalar k
  __shared__ int qt_s[KC][NWC];             // offset of its source node inside a tile element
  __shared__ int qh_s[KC];                  // offset inside a tile element's halo block
  // per-stage tile metadata, written by the producer before its release-arrive
  __shared__ long long me0_s[NS];
  __shared__ int mnt_s[NS], mfast_s[NS];
  __shared__ unsigned mcset_s[NS];          // classes present in the tile (bit set)
  __shared__ int mmask_s[NS][E], mcls_s[NS][E];
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
  for (int i = tid; i < N1 * N1; i += blockDim.x) {
    chol_s[i] = a.chol1d[i];
    const int ia = i / N1, k = i % N1;
    cshift_s[i] = (ia + k < N1) ? a.chol1d[(ia + k) * N1 + ia] : 0.0;
  }
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
      mbar_init(&full_bar[s], 1 + 32);
      mbar_init(&empty_bar[s], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const int fast_class = a.class_of_mask[0];
  const int ntiles = (int)geo.ntiles;

  if (tid >= NC) {
    // ============================ producer warp ============================
    const int lane = tid - NC;
    const int c0 = (int)a.g.cells[0];
    const int per0 = a.g.periodic[0];
    const int nlay = (int)(a.g.layer_end - a.g.layer_begin);
    const int lsi = (int)ls;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int stage = it % NS;
      if (it >= NS) mbar_wait(&empty_bar[stage], ((it / NS) - 1) & 1);
      double* sst = sm + stage * C::STAGE;
      double* ust = sst + TILE;
      double* hst = ust + TILE;
      STile<D> ti;
      ti.init(a.g, tile, E, nlay, lsi);
      const int e0 = ti.e0;
      const int nt = ti.nt;
      // tile metadata for the consumers (mask of missing neighbours, class)
      int cls = -1;
      if (lane < E) {
        const int mask = ti.mask(lane, c0, per0);
        cls = a.class_of_mask[mask];
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
      }
      __syncwarp();
      if (lane == 0) {
        const uint32_t bytes = (uint32_t)(nt * NV * sizeof(double));
        mbar_arrive_expect_tx(&full_bar[stage], 2 * bytes);  // release: metadata above
        bulk_g2s(sst, a.s + (int64_t)e0 * NV, bytes, &full_bar[stage]);
        bulk_g2s(ust, uo + (int64_t)e0 * NV, bytes, &full_bar[stage]);
      }
      // neighbour face nodes not inside the tile, as runs of face nodes
      // (consecutive lanes -> consecutive nodes: coalesced 8-byte cp.async)
      constexpr int RUN = NWC * NF;
#pragma unroll
      for (int ci = 0; ci < NCF; ++ci) {
        const int f = cf_s[ci];
        if ((f >> 1) == 0) {
          const int t = (f == 0) ? 0 : nt - 1;
          const int i = ti.i0 + t;
          const bool ex = (f == 0) ? (i > 0 || per0) : (i < c0 - 1 || per0);
          if (!ex) continue;
          const int nb = e0 + t + ((f == 0) ? (i > 0 ? -1 : c0 - 1) : (i < c0 - 1 ? 1 : -(c0 - 1)));
          const double* base = uo + (int64_t)nb * NV;
          for (int item = lane; item < RUN; item += 32) {
            const int j = item / NF, n = item - (item / NF) * NF;
            cp_async8(hst + ((t * NCF + ci) * NWC + j) * NF + n, base + wc_s[ci][j] * NP + fv_s[f ^ 1][n]);
          }
        } else {
          if (!ti.face_has(f)) continue;
          const double* base = uo + ((int64_t)e0 + ti.face_off(f)) * NV;
          for (int item = lane; item < nt * RUN; item += 32) {
            const int t = item / RUN;
            const int rem = item - t * RUN;
            const int j = rem / NF, n = rem - j * NF;
            cp_async8(hst + ((t * NCF + ci) * NWC + j) * NF + n,
                      base + t * NV + wc_s[ci][j] * NP + fv_s[f ^ 1][n]);
          }
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
    // DMMA A fragments of the interior-class operator for this warp's row
    // tiles: Lf[j][ks] = L[8 rt_j + (lane>>2)][4 ks + (lane&3)]
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
    // C fragments for the 2D tensor-core norm: C[4 ks + (lane&3)][lane>>2]
    double cfr[2];
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int kk = 4 * ks + (lane & 3), nn = lane >> 2;
      cfr[ks] = (kk < N1 && nn < N1) ? chol_s[kk * N1 + nn] : 0.0;
    }
    // per-thread constants of the DFMA (3D) norm: row r, node indices
    const int rr = rv ? r : 0;
    const double cw = rv ? a.comp_w[rr / NP] * a.jac : 0.0;
    int ia_ax[D];
    {
      int mul = 1;
#pragma unroll
      for (int ax = 0; ax < D; ++ax) {
        ia_ax[ax] = ((rr % NP) / mul) % N1;
        mul *= N1;
      }
    }

    int it = 0;
    int prev_tile = -1;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int stage = it % NS;
      const int ob = it & 1;
      mbar_wait(&full_bar[stage], (it / NS) & 1);
      if (tid == 0 && it >= 2) bulk_wait_read<1>();   // out[ob] free again
      const int e0 = (int)me0_s[stage];
      const int nt = mnt_s[stage];
      const int fast = mfast_s[stage];
      const double* sst = sm + stage * C::STAGE;
      const double* ust = sst + TILE;
      const double* hst = ust + TILE;
      // ---- neighbour face scalars q[t][k] (TraceSnapshot of iterate k) ----
#pragma unroll
      for (int m = 0; m < (E * KC + NC - 1) / NC; ++m) {
        const int idx = tid + m * NC;
        if (idx < E * KC) {
          const int t = idx / KC, k = idx - (idx / KC) * KC;
          const int f = qf_s[k];
          double v = 0.0;
          if (!(mmask_s[stage][t] & (1 << f))) {
            const bool in_tile = (f >> 1) == 0 && !((f == 0 && t == 0) || (f == 1 && t == nt - 1));
            const int ci = k / NF;
            if (in_tile) {
              const double* src = ust + (t + (f == 0 ? -1 : 1)) * NV;
#pragma unroll
              for (int j = 0; j < NWC; ++j) v = fma(ww_s[ci][j], src[qt_s[k][j]], v);
            } else {
              const double* src = hst + t * (NCF * NWC * NF) + qh_s[k];
#pragma unroll
              for (int j = 0; j < NWC; ++j) v = fma(ww_s[ci][j], src[j * NF], v);
            }
          }
          q_s[idx] = v;
        }
      }
      consumer_bar(NC);
      double* outb = out_s + ob * TILE;
      double* dcur = C::PIPE ? d_s + (it & 1) * TILE : d_s;
      // ---- (PIPE) norm of the previous tile, independent of the DMMAs below
      double nsum = 0.0;
      if constexpr (C::PIPE) {
        if (it > 0)
          nsum = norm_units_2d<N1, M, NP, NV, E, NCW, UPW>(d_s + ((it - 1) & 1) * TILE, warp, lane, cfr,
                                                           a.comp_w);
      }
      // ---- lifted local solve u^{k+1} = s + L q on the fp64 tensor core --
      // D[row][elem] = s + sum_k L[row][k] q[elem][k]: rows = 8 x NRT row
      // tiles (warp w owns tiles w, w+NCW, ...), elements = 8 x NEG groups.
      double acc[NEG][RTW][2];
#pragma unroll
      for (int eg = 0; eg < NEG; ++eg) {
        const int te = eg * 8 + 2 * (lane & 3);   // D columns (elements) of this lane
#pragma unroll
        for (int j = 0; j < RTW; ++j) {
          const int row = (warp + j * NCW) * 8 + (lane >> 2);
          const bool ok = row < NV && (warp + j * NCW) < NRT;
          acc[eg][j][0] = ok ? sst[te * NV + row] : 0.0;
          acc[eg][j][1] = ok ? sst[(te + 1) * NV + row] : 0.0;
        }
      }
      const double* qb = q_s + (lane >> 2) * KC + (lane & 3);
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
        // one masked pass per operator class present in the tile
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
              const double b = (mcls_s[stage][eg * 8 + (lane >> 2)] == c) ? qb[eg * 8 * KC + 4 * ks] : 0.0;
#pragma unroll
              for (int j = 0; j < RTW; ++j) dmma_8x8x4(acc[eg][j][0], acc[eg][j][1], av[j], b);
            }
          }
        }
      }
#pragma unroll
      for (int eg = 0; eg < NEG; ++eg) {
        const int te = eg * 8 + 2 * (lane & 3);
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
      if constexpr (C::PIPE) {
        if (it > 0) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, o);
          if (lane == 0) red_s[((it - 1) & 1) * 32 + warp] = nsum;
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[stage]);
      consumer_bar(NC);
      if (tid == 0) {
        bulk_s2g(un + (int64_t)e0 * NV, outb, (uint32_t)(nt * NV * sizeof(double)));
        bulk_commit();
        if (C::PIPE && it > 0) {
          double s = 0.0;
          for (int w = 0; w < NCW; ++w) s += red_s[((it - 1) & 1) * 32 + w];
          a.tile_partials[prev_tile] = a.jac * s;
        }
      }
      if constexpr (!C::PIPE) {
        // ---- ||delta||_M^2 by sum-factorised Cholesky passes (C^T per axis)
        double* src = d_s;
        double* dst = t_s;
        double acc2 = 0.0;
        int mul = 1;
#pragma unroll
        for (int ax = 0; ax < D; ++ax) {
          const bool last_ax = ax == D - 1;
          const int ia = ia_ax[ax];
          const double* cw_row = cshift_s + ia * N1;
#pragma unroll
          for (int tt = 0; tt < EG; ++tt) {
            const int t = g * EG + tt;
            const double* p = src + t * NV + rr;
            double v = 0.0;
#pragma unroll
            for (int k = 0; k < N1; ++k) v = fma(cw_row[k], p[(ia + k < N1) ? k * mul : 0], v);
            if (last_ax) acc2 = fma(v, v, acc2);
            else if (rv) dst[t * NV + r] = v;
          }
          if (!last_ax) {
            consumer_bar(NC);
            double* tmp = src;
            src = dst;
            dst = tmp;
          }
          mul *= N1;
        }
        double tsum = rv ? cw * acc2 : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
        if (lane == 0) red_s[warp] = tsum;
        consumer_bar(NC);
        if (tid == 0) {
          double s = 0.0;
          for (int w = 0; w < NCW; ++w) s += red_s[w];
          a.tile_partials[tile] = s;
        }
      }
      prev_tile = tile;
    }
    if constexpr (C::PIPE) {
      // drain: norm of the last tile
      if (it > 0) {
        double nsum = norm_units_2d<N1, M, NP, NV, E, NCW, UPW>(d_s + ((it - 1) & 1) * TILE, warp, lane, cfr,
                                                                a.comp_w);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, o);
        if (lane == 0) red_s[((it - 1) & 1) * 32 + warp] = nsum;
        consumer_bar(NC);
        if (tid == 0) {
          double s = 0.0;
          for (int w = 0; w < NCW; ++w) s += red_s[((it - 1) & 1) * 32 + w];
          a.tile_partials[prev_tile] = a.jac * s;
        }
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
      int64_t n_rows, row_len;
      partial_rows(geo, n_rows, row_len);
      finalize_block(a.tile_partials, n_rows, row_len, st, a.norm_hist);
    }
  }
}

}  // namespace ihdg
