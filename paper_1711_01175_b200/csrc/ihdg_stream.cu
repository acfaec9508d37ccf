// Instantiations + dispatch of the streaming sweep kernels (k_sweep_ws,
// k_sweep_v3, k_sweep_v4).  Which kernel a call uses is decided here from
// the args (stream_entry) and the process-wide selector set by
// ihdg_set_sweep_impl; ihdg_sweep_kernel reports the decision by name.
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ihdg_stream.cuh"
#include "ihdg_ws.cuh"
#include "ihdg_v3.cuh"
#include "ihdg_v4.cuh"
#include "ihdg_gemv.cuh"
#include "ihdg_v5.cuh"

namespace ihdg {

// IHDG_NO_PDL=1 turns programmatic dependent launch off (A/B)
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("IHDG_NO_PDL");
    return !(e != nullptr && e[0] == '1');
  }();
  return on;
}

// Launch one persistent grid (one CTA per SM) of kernel K with BYTES of
// dynamic shared memory; the attribute is set once per device.
template <auto kernel>
cudaError_t launch_persistent(int nt, size_t bytes, int tile_elems, const ihdg_sweep_args* a, cudaStream_t st,
                              bool cooperative = false, int ctas_per_sm = 1, bool pdl = true) {
  static std::atomic<unsigned> configured{0u};   // per kernel: bit per device ordinal (< 32)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned bit = 1u << (dev & 31);
  if ((configured.load() & bit) == 0u) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit);
  }
  int sms = 0;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  Geo geo;
  geo.init(a->g, tile_elems);
  sms *= ctas_per_sm;
  int64_t grid = geo.ntiles < sms ? geo.ntiles : sms;
  if (grid < 1) grid = 1;
  if (cooperative) {
    // co-residency of the whole grid is guaranteed (or the launch fails):
    // the kernel's grid barrier cannot deadlock
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, *a);
  }
  if (pdl && pdl_enabled()) {
    // programmatic dependent launch: the prologue of this sweep (tables, L
    // fragments, barriers) overlaps the tail of the previous launch in the
    // stream; the kernel waits (griddepcontrol.wait) before it touches data
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, *a);
  }
  kernel<<<(unsigned)grid, nt, bytes, st>>>(*a);
  return cudaGetLastError();
}

template <int N1, int M, int NCF, int NWC, int E, int NS>
cudaError_t launch_ws_t(const ihdg_sweep_args* a, cudaStream_t st) {
  static_assert(E == Cfg<2, N1, M>::TE, "ws tile must equal the generic tile (tile partial count)");
  const bool coop = a->finalize && a->layer_sums != nullptr && a->grid_bar != nullptr;   // parallel finalize
  if (a->q_store != nullptr && a->gram_kc == NCF * N1) {   // Gram-form norm instantiation
    using C = WCfg<N1, M, NCF, NWC, E, NS, true>;
    return launch_persistent<k_sweep_ws<N1, M, NCF, NWC, E, NS, true>>(C::NT, C::BYTES, E, a, st, coop);
  }
  using C = WCfg<N1, M, NCF, NWC, E, NS, false>;
  return launch_persistent<k_sweep_ws<N1, M, NCF, NWC, E, NS, false>>(C::NT, C::BYTES, E, a, st, coop);
}

template <int D, int N1, int M, int NCF, int NWC, int NS, int NCW, int PF, int NQW>
cudaError_t launch_v3_t(const ihdg_sweep_args* a, cudaStream_t st) {
  using C = V3Cfg<D, N1, M, NCF, NWC, NS, NCW, PF, NQW>;
  static_assert(8 * PF == Cfg<D, N1, M>::TE, "v3 logical tile must equal the generic tile (tile partial count)");
  return launch_persistent<k_sweep_v3<D, N1, M, NCF, NWC, NS, NCW, PF, NQW>>(C::NT, C::BYTES, 8 * PF, a, st);
}

template <int FMASK, int NW, int MINB>
cudaError_t launch_v4_t(const ihdg_sweep_args* a, cudaStream_t st) {
  using C = V4Cfg<FMASK, NW, MINB>;
  static_assert(8 * C::PF == Cfg<3, 4, 1>::TE, "v4 logical tile must equal the generic tile (tile partial count)");
  return launch_persistent<k_sweep_v4<FMASK, NW, MINB>>(C::NT, C::BYTES, 8 * C::PF, a, st, false, MINB);
}

// per-element operators (GEMV mode): as many CTAs per SM as fit, one tile each
template <int D, int N1, int M>
cudaError_t launch_gemv_t(const ihdg_sweep_args* a, cudaStream_t st) {
  using G = GCfg<D, N1, M>;
  static std::atomic<int> cps{0};   // resident CTAs per SM (same for every device of one model)
  int c = cps.load();
  if (c == 0) {
    cudaError_t e = cudaFuncSetAttribute(k_sweep_gemv<D, N1, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::BYTES);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, k_sweep_gemv<D, N1, M>, G::NT, G::BYTES);
    if (e != cudaSuccess) return e;
    if (c < 1) c = 1;
    cps.store(c);
  }
  // no programmatic dependent launch here: with three CTAs per SM the next
  // grid's CTAs settle early on the free slots and skew the placement
  // (measured 0.087 -> 0.090 ms at 16^3 p=2)
  return launch_persistent<k_sweep_gemv<D, N1, M>>(G::NT, G::BYTES, G::TE, a, st, false, c, false);
}

template <int N1, int M, int NWC, int NW, int PF>
cudaError_t launch_v5_t(const ihdg_sweep_args* a, cudaStream_t st) {
  using C = V5Cfg<N1, M, NWC, NW, PF>;
  static_assert(8 * PF == Cfg<2, N1, M>::TE, "v5 logical tile must equal the generic tile (tile partial count)");
  return launch_persistent<k_sweep_v5<N1, M, NWC, NW, PF>>(C::NT, C::BYTES, 8 * PF, a, st);
}

enum Kind { KIND_V3 = 0, KIND_WS = 1, KIND_V4 = 2, KIND_GEMV = 3, KIND_V5 = 4 };
const char* const kKindName[] = {"k_sweep_v3", "k_sweep_ws", "k_sweep_v4", "k_sweep_gemv", "k_sweep_v5"};

struct StreamEntry {
  int D, N1, M, NCF, NWC, E, NV;
  cudaError_t (*launch)(const ihdg_sweep_args*, cudaStream_t);
  int kind;
  int fmask = -1;   // >= 0: the entry needs exactly this set of coupled faces
};

#define IHDG_V3(D, N1, M, NCF, NWC, NS, NCW, PF, NQW) \
  {D, N1, M, NCF, NWC, 8 * PF, M * Pow<N1, D>::v, launch_v3_t<D, N1, M, NCF, NWC, NS, NCW, PF, NQW>, KIND_V3},
#define IHDG_V4(FMASK, NW, MINB) {3, 4, 1, v4_popc(FMASK), 1, 32, 64, launch_v4_t<FMASK, NW, MINB>, KIND_V4, FMASK},
#define IHDG_V5(N1, M, NWC, NW, PF) {2, N1, M, 4, NWC, 8 * PF, M * N1 * N1, launch_v5_t<N1, M, NWC, NW, PF>, KIND_V5},
#define IHDG_WS(N1, M, NCF, NWC, E, NS) \
  {2, N1, M, NCF, NWC, E, M * N1 * N1, launch_ws_t<N1, M, NCF, NWC, E, NS>, KIND_WS},

#ifndef IHDG_WS5_NS
#define IHDG_WS5_NS 3   // stage count of the config-5 ring (A/B builds override it)
#endif
// config-4 v3 shape (A/B builds override it): stages, consumer warps, prep warps
#ifndef IHDG_C4_NS
#define IHDG_C4_NS 10
#endif
#ifndef IHDG_C4_NCW
#define IHDG_C4_NCW 7
#endif
#ifndef IHDG_C4_NQW
#define IHDG_C4_NQW 8
#endif
// configs 2/3 v3 shape (A/B builds override it)
#ifndef IHDG_C23_NS
#define IHDG_C23_NS 16
#endif
#ifndef IHDG_C23_NCW
#define IHDG_C23_NCW 7
#endif
#ifndef IHDG_C23_NQW
#define IHDG_C23_NQW 8
#endif

// config-4 v4 shape (A/B builds override it): warps per CTA, CTAs per SM
#ifndef IHDG_C4_V4_NW
#define IHDG_C4_V4_NW 16
#endif
#ifndef IHDG_C4_V4_MINB
#define IHDG_C4_V4_MINB 1
#endif

// First match wins: v4 before v3 before ws for the same (D, N1, M).
const StreamEntry kStream[] = {
#ifndef IHDG_NO_V5
    IHDG_V5(5, 3, 2, 16, 2)   // configs 2/3: CD / SW 2D p=4, register-tiled
#endif
    // config 4: transport 3D p=3; one instantiation per inflow-face set (the
    // sign pattern of beta; config 4 itself is faces 0, 2, 4 = 0x15)
    IHDG_V4(0x15, IHDG_C4_V4_NW, IHDG_C4_V4_MINB) IHDG_V4(0x16, IHDG_C4_V4_NW, IHDG_C4_V4_MINB)
    IHDG_V4(0x19, IHDG_C4_V4_NW, IHDG_C4_V4_MINB) IHDG_V4(0x1a, IHDG_C4_V4_NW, IHDG_C4_V4_MINB)
    IHDG_V4(0x25, IHDG_C4_V4_NW, IHDG_C4_V4_MINB) IHDG_V4(0x26, IHDG_C4_V4_NW, IHDG_C4_V4_MINB)
    IHDG_V4(0x29, IHDG_C4_V4_NW, IHDG_C4_V4_MINB) IHDG_V4(0x2a, IHDG_C4_V4_NW, IHDG_C4_V4_MINB)
    IHDG_V3(2, 5, 3, 4, 2, IHDG_C23_NS, IHDG_C23_NCW, 2, IHDG_C23_NQW)  // configs 2/3: CD / SW 2D p=4
    IHDG_V3(3, 4, 1, 3, 1, IHDG_C4_NS, IHDG_C4_NCW, 4, IHDG_C4_NQW)  // config 4: transport 3D p=3
    IHDG_WS(7, 3, 4, 2, 16, IHDG_WS5_NS)   // config 5: CD 2D p=6 (warp-specialised)
    IHDG_WS(5, 3, 4, 2, 16, 4)             // configs 2/3 without v3
};

// Per-element operators with raw neighbour values (GEMV mode), by (D, N1, M):
// the elements large enough to keep a CTA of row threads busy (NV >= 108;
// measured on B200, cdr_manufactured: 16^3 p=2 0.267 -> 0.105 ms, 8^3 p=3
// 0.244 -> 0.083 ms, but 16^3 p=1 (NV = 32, one consumer warp) 0.068 -> 0.225 ms,
// so the small ones stay on the generic kernel).
#define IHDG_GEMV(D, N1, M) {D, N1, M, 0, 0, Cfg<D, N1, M>::TE, M * Pow<N1, D>::v, launch_gemv_t<D, N1, M>, KIND_GEMV},
const StreamEntry kGemv[] = {
    IHDG_GEMV(3, 3, 4) IHDG_GEMV(3, 4, 4) IHDG_GEMV(3, 5, 4)   // cdr_manufactured (3D, variable beta) p = 2..4
};

// Process-wide kernel selector (ihdg_set_sweep_impl); the initial value comes
// from IHDG_SWEEP_IMPL so A/B tools keep working.
enum Impl { IMPL_AUTO = 0, IMPL_NO_V3 = 1, IMPL_GENERIC = 2, IMPL_V3 = 3, IMPL_V5 = 4 };
std::atomic<int> g_impl{-1};

int parse_impl(const char* s) {
  if (s == nullptr || s[0] == '\0' || std::strcmp(s, "auto") == 0) return IMPL_AUTO;
  if (std::strcmp(s, "ws") == 0 || std::strcmp(s, "stream") == 0) return IMPL_NO_V3;
  if (std::strcmp(s, "generic") == 0) return IMPL_GENERIC;
  if (std::strcmp(s, "v3") == 0) return IMPL_V3;   // skip v4 / v5
  if (std::strcmp(s, "v5") == 0) return IMPL_V5;   // v5 wherever it applies (no round model)
  return -1;
}

int current_impl() {
  int v = g_impl.load();
  if (v < 0) {
    const int e = parse_impl(std::getenv("IHDG_SWEEP_IMPL"));
    v = e < 0 ? IMPL_AUTO : e;
    int expect = -1;
    g_impl.compare_exchange_strong(expect, v);
    v = g_impl.load();
  }
  return v;
}

// k_sweep_v5 or k_sweep_v3 for a 2D p=4 strip?  Both walk 8-element tiles in
// rounds (v5: 16 warps per SM, one tile each; v3: 7 consumer warps per SM), so
// the sweep time is a fixed part plus rounds x time per round.  Measured on
// B200 (us; profiles/r02_v5_ab.txt): v5 9.2 + 9.3 rounds, v3 15.6 + 3.4 rounds:
// v5 wins where its rounds are well filled (config 2: 2048 tiles, one round),
// v3 on config 3 (8192 tiles: 3.46 -> 4 rounds of v5 against 7.9 -> 8 of v3).
bool v5_cheaper(const ihdg_geom& g) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  Geo geo;
  geo.init(g, 8);
  const double tiles = (double)geo.ntiles;
  const double r5 = std::ceil(tiles / (16.0 * sms)), r3 = std::ceil(tiles / (7.0 * sms));
  if (r3 < 2.0) return false;   // one round of v3 (up to ~96^2): its floor is lower (16^2: 9-12 us against 14-17 us)
  return 9.2 + 9.3 * r5 < 15.6 + 3.4 * r3;
}

// Returns the entry usable for these args, or nullptr (generic kernel).
const StreamEntry* stream_entry(const ihdg_sweep_args* a) {
  const int impl = current_impl();
  if (impl == IMPL_GENERIC) return nullptr;
  if (a->norm_kind != IHDG_NORM_VOLUME) return nullptr;
  if (a->per_element && (a->raw_blocks == 2 || a->raw_blocks == 4)) {   // per-element operators: GEMV kernel
    const ihdg_geom& gg = a->g;
    for (const StreamEntry& e : kGemv) {
      if (e.D != gg.dim || e.N1 != gg.order + 1 || e.M != gg.ncomp) continue;
      if (((uintptr_t)a->LT) % 16 != 0) continue;   // bulk copies of the operator chunks
      Geo geo;
      geo.init(gg, e.E);
      if (geo.nloc + 2 * geo.ls >= (1LL << 31)) continue;   // 32-bit element indices
      return &e;
    }
    return nullptr;
  }
  if (a->per_element || a->raw_blocks > 0) return nullptr;   // other per-element layouts: generic kernel
  if (a->scheme != IHDG_SCHEME_II) return nullptr;   // iHDG-I: generic kernel
  const ihdg_geom& g = a->g;
  int ncf = 0, maxw = 0, fmask = 0;
  for (int f = 0; f < 2 * g.dim; ++f) {
    if (!a->coupled[f]) continue;
    ++ncf;
    fmask |= 1 << f;
    int w = 0;
    for (int c = 0; c < g.ncomp; ++c) w += a->face_w[f][c] != 0.0;
    maxw = w > maxw ? w : maxw;
  }
  for (const StreamEntry& e : kStream) {
    if (e.D != g.dim || e.N1 != g.order + 1 || e.M != g.ncomp) continue;
    if (e.NCF != ncf || maxw > e.NWC) continue;
    if (e.fmask >= 0 && e.fmask != fmask) continue;
    if ((e.kind == KIND_V3 || e.kind == KIND_V4 || e.kind == KIND_V5) && impl == IMPL_NO_V3) continue;
    if ((e.kind == KIND_V4 || e.kind == KIND_V5) && impl == IMPL_V3) continue;
    if (e.kind == KIND_V5 && impl != IMPL_V5 && !v5_cheaper(g)) continue;
    Geo geo;
    geo.init(g, e.E);
    if (geo.tile_len % e.E != 0) continue;                       // full tiles only
    if (g.cells[0] % ((e.kind == KIND_V3 || e.kind == KIND_V4 || e.kind == KIND_V5) ? 8 : e.E) != 0) continue;  // tiles inside one axis-0 row
    if (geo.nloc + 2 * geo.ls >= (1LL << 31) || geo.ntiles >= (1LL << 31)) continue;  // 32-bit indices
    if ((geo.ls * e.NV * 8) % 16 != 0) continue;                  // ghost offset
    if (((uintptr_t)a->u_old | (uintptr_t)a->u_new | (uintptr_t)a->s) % 16 != 0) continue;
    return &e;
  }
  return nullptr;
}

}  // namespace ihdg

#ifdef IHDG_WS_PROF
// profiling build only: read (and optionally reset) the per-role counters
extern "C" int ihdg_ws_prof(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, ihdg::g_ws_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(ihdg::g_ws_prof, z, sizeof(z));
  }
  return 0;
}
#endif

#ifdef IHDG_WS_TRACE
// trace build only: the phase timestamps of CTA 0 (tools/ws_trace.py)
extern "C" int ihdg_ws_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, ihdg::g_ws_trace, sizeof(long long) * 16 * 8 * 12);
}
#endif

// 1 if the streaming kernel is used for these args, 0 for the generic one.
int ihdg_stream_variant(const ihdg_sweep_args* a) { return ihdg::stream_entry(a) != nullptr ? 1 : 0; }

// Name of the streaming kernel these args dispatch to, or nullptr (generic).
const char* ihdg_stream_kernel_name(const ihdg_sweep_args* a) {
  const ihdg::StreamEntry* e = ihdg::stream_entry(a);
  return e == nullptr ? nullptr : ihdg::kKindName[e->kind];
}

// Gram-form norm columns (q scalars per element) of the kernel these args
// dispatch to: k_sweep_ws only (ihdg.h, ihdg_sweep_args.q_store)
int ihdg_stream_gram_kc(const ihdg_sweep_args* a) {
  const ihdg::StreamEntry* e = ihdg::stream_entry(a);
  if (e == nullptr || e->kind != ihdg::KIND_WS) return 0;
  return e->NCF * e->N1;
}

// 0 ok, -1 unknown name
int ihdg_stream_set_impl(const char* name) {
  const int v = ihdg::parse_impl(name);
  if (v < 0) return -1;
  ihdg::g_impl.store(v);
  return 0;
}

// Launch the streaming kernel if applicable. Returns 1 launched, 0 not
// applicable, -1 on a launch error (*err holds it).
int ihdg_stream_launch(const ihdg_sweep_args* a, cudaStream_t st, cudaError_t* err) {
  const ihdg::StreamEntry* e = ihdg::stream_entry(a);
  if (e == nullptr) return 0;
  const cudaError_t rc = e->launch(a, st);
  if (rc != cudaSuccess) {
    if (err) *err = rc;
    return -1;
  }
  return 1;
}
