// Shared device helpers of the streaming sweep kernels (k_sweep_ws,
// k_sweep_v3, k_sweep_v4) for sm_100a: mbarrier / TMA bulk-copy / DMMA
// wrappers, the 32-bit tile geometry (STile, FastDiv) and the optional per-role
// cycle counters of the profiling build.
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

// Timeline trace of CTA 0 (trace build, -DIHDG_WS_TRACE; tools/ws_trace.py):
// lane 0 of every warp stamps clock64 at its phase boundaries for iterations
// IHDG_TRACE_IT0 .. +7
#ifdef IHDG_WS_TRACE
#ifndef IHDG_TRACE_IT0
#define IHDG_TRACE_IT0 400
#endif
__device__ long long g_ws_trace[16][8][12];
#define WS_STAMP(warp, it, slot)                                                              \
  do {                                                                                        \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0 && (it) >= IHDG_TRACE_IT0 && (it) < IHDG_TRACE_IT0 + 8) \
      g_ws_trace[warp][(it) - IHDG_TRACE_IT0][slot] = clock64();                              \
  } while (0)
#else
#define WS_STAMP(warp, it, slot)
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
// Programmatic dependent launch (launch attribute
// cudaLaunchAttributeProgrammaticStreamSerialization): a sweep lets the next
// launch in the stream start its prologue early, and every sweep waits for
// the previous grid to complete (and flush) before it reads anything the
// previous grid wrote.  Both are no-ops without the launch attribute.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
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

}  // namespace ihdg
