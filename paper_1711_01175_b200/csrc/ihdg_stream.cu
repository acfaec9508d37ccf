// Instantiations + dispatch of the streaming sweep (ihdg_stream.cuh).
#include <cstdlib>
#include <cstring>
#include <string>

#include "ihdg_stream.cuh"
#include "ihdg_ws.cuh"
#include "ihdg_v3.cuh"
#include "ihdg_ws2.cuh"
#include "ihdg_ws3.cuh"
#include "ihdg_ws4.cuh"

namespace ihdg {

int stream_sms() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

template <int D, int N1, int M, int NCF, int NWC, int E, int NS, int G>
int launch_stream_t(const ihdg_sweep_args* a, cudaStream_t st) {
  using C = SCfg<D, N1, M, NCF, NWC, E, NS, G>;
  static_assert(E == Cfg<D, N1, M>::TE, "stream tile must equal the generic tile (tile partial count)");
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_sweep_stream<D, N1, M, NCF, NWC, E, NS, G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
    if (e != cudaSuccess) return -2;
    configured = true;
  }
  Geo geo;
  geo.init(a->g, E);
  int64_t grid = geo.ntiles < stream_sms() ? geo.ntiles : stream_sms();
  if (grid < 1) grid = 1;
  k_sweep_stream<D, N1, M, NCF, NWC, E, NS, G><<<(unsigned)grid, C::NT, C::BYTES, st>>>(*a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

template <int N1, int M, int NCF, int NWC, int E, int NS>
int launch_ws3_t(const ihdg_sweep_args* a, cudaStream_t st) {
  using C = W3Cfg<N1, M, NCF, NWC, E, NS>;
  static_assert(E == Cfg<2, N1, M>::TE, "ws3 tile must equal the generic tile (tile partial count)");
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_sweep_ws3<N1, M, NCF, NWC, E, NS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
    if (e != cudaSuccess) return -2;
    configured = true;
  }
  Geo geo;
  geo.init(a->g, E);
  int64_t grid = geo.ntiles < stream_sms() ? geo.ntiles : stream_sms();
  if (grid < 1) grid = 1;
  k_sweep_ws3<N1, M, NCF, NWC, E, NS><<<(unsigned)grid, C::NT, C::BYTES, st>>>(*a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

template <int N1, int M, int NCF, int NWC, int NS>
int launch_ws4_t(const ihdg_sweep_args* a, cudaStream_t st) {
  using C = W4Cfg<N1, M, NCF, NWC, NS>;
  static_assert(C::EL == Cfg<2, N1, M>::TE, "ws4 logical tile must equal the generic tile (tile partial count)");
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_sweep_ws4<N1, M, NCF, NWC, NS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
    if (e != cudaSuccess) return -2;
    configured = true;
  }
  Geo geo;
  geo.init(a->g, C::EL);
  int64_t grid = geo.ntiles < stream_sms() ? geo.ntiles : stream_sms();
  if (grid < 1) grid = 1;
  k_sweep_ws4<N1, M, NCF, NWC, NS><<<(unsigned)grid, C::NT, C::BYTES, st>>>(*a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

template <int N1, int M, int NCF, int NWC, int E, int NS>
int launch_ws_t(const ihdg_sweep_args* a, cudaStream_t st) {
  using C = WCfg<N1, M, NCF, NWC, E, NS>;
  static_assert(E == Cfg<2, N1, M>::TE, "ws tile must equal the generic tile (tile partial count)");
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_sweep_ws<N1, M, NCF, NWC, E, NS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
    if (e != cudaSuccess) return -2;
    configured = true;
  }
  Geo geo;
  geo.init(a->g, E);
  int64_t grid = geo.ntiles < stream_sms() ? geo.ntiles : stream_sms();
  if (grid < 1) grid = 1;
  k_sweep_ws<N1, M, NCF, NWC, E, NS><<<(unsigned)grid, C::NT, C::BYTES, st>>>(*a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

template <int D, int N1, int M, int NCF, int NWC, int NS, int NCW, int PF, int NQW>
int launch_v3_t(const ihdg_sweep_args* a, cudaStream_t st) {
  using C = V3Cfg<D, N1, M, NCF, NWC, NS, NCW, PF, NQW>;
  static_assert(8 * PF == Cfg<D, N1, M>::TE, "v3 logical tile must equal the generic tile (tile partial count)");
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_sweep_v3<D, N1, M, NCF, NWC, NS, NCW, PF, NQW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
    if (e != cudaSuccess) return -2;
    configured = true;
  }
  Geo geo;
  geo.init(a->g, 8 * PF);
  int64_t grid = geo.ntiles < stream_sms() ? geo.ntiles : stream_sms();
  if (grid < 1) grid = 1;
  k_sweep_v3<D, N1, M, NCF, NWC, NS, NCW, PF, NQW><<<(unsigned)grid, C::NT, C::BYTES, st>>>(*a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

template <int N1, int M, int NCF, int NWC, int E, int NS>
int launch_ws2_t(const ihdg_sweep_args* a, cudaStream_t st) {
  using C = W2Cfg<N1, M, NCF, NWC, E, NS>;
  static_assert(E == Cfg<2, N1, M>::TE, "ws2 tile must equal the generic tile (tile partial count)");
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k_sweep_ws2<N1, M, NCF, NWC, E, NS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::BYTES);
    if (e != cudaSuccess) return -2;
    configured = true;
  }
  Geo geo;
  geo.init(a->g, E);
  int64_t grid = geo.ntiles < stream_sms() ? geo.ntiles : stream_sms();
  if (grid < 1) grid = 1;
  k_sweep_ws2<N1, M, NCF, NWC, E, NS><<<(unsigned)grid, C::NT, C::BYTES, st>>>(*a);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

struct StreamEntry {
  int D, N1, M, NCF, NWC, E, NV;
  int (*launch)(const ihdg_sweep_args*, cudaStream_t);
  int v3;  // version-3 kernel (physical 8-element tiles)
  int ws3; // opt-in kernels: 1 k_sweep_ws3 (IHDG_SWEEP_IMPL=ws3), 2 k_sweep_ws4 (=ws4), 3 k_sweep_v3 on config 5 (=v3)
};

#define IHDG_V3(D, N1, M, NCF, NWC, NS, NCW, PF, NQW) \
  {D, N1, M, NCF, NWC, 8 * PF, M * Pow<N1, D>::v, launch_v3_t<D, N1, M, NCF, NWC, NS, NCW, PF, NQW>, 1, 0},
#define IHDG_WS2(N1, M, NCF, NWC, E, NS) \
  {2, N1, M, NCF, NWC, E, M * N1 * N1, launch_ws2_t<N1, M, NCF, NWC, E, NS>, 0, 0},
#ifndef IHDG_WS5_NS
#define IHDG_WS5_NS 3   // stage count of the config-5 ring (A/B builds override it)
#endif
#define IHDG_WS(N1, M, NCF, NWC, E, NS) \
  {2, N1, M, NCF, NWC, E, M * N1 * N1, launch_ws_t<N1, M, NCF, NWC, E, NS>, 0, 0},
#ifndef IHDG_WS4_NS
#define IHDG_WS4_NS 6
#endif
#ifndef IHDG_WS3_NS
#define IHDG_WS3_NS 3
#endif
#define IHDG_WS3(N1, M, NCF, NWC, E, NS) \
  {2, N1, M, NCF, NWC, E, M * N1 * N1, launch_ws3_t<N1, M, NCF, NWC, E, NS>, 0, 1},
#define IHDG_STREAM(D, N1, M, NCF, NWC, E, NS, G) \
  {D, N1, M, NCF, NWC, E, M * Pow<N1, D>::v, launch_stream_t<D, N1, M, NCF, NWC, E, NS, G>, 0, 0},

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

// config-5 v3 (opt-in, IHDG_SWEEP_IMPL=v3) shape
#ifndef IHDG_C5V3_NS
#define IHDG_C5V3_NS 16
#endif
#ifndef IHDG_C5V3_NCW
#define IHDG_C5V3_NCW 7
#endif
#ifndef IHDG_C5V3_NQW
#define IHDG_C5V3_NQW 8
#endif

const StreamEntry kStream[] = {
    IHDG_V3(2, 5, 3, 4, 2, IHDG_C23_NS, IHDG_C23_NCW, 2, IHDG_C23_NQW)  // configs 2/3: CD / SW 2D p=4
    IHDG_V3(3, 4, 1, 3, 1, IHDG_C4_NS, IHDG_C4_NCW, 4, IHDG_C4_NQW)  // config 4: transport 3D p=3
    IHDG_WS2(7, 3, 4, 2, 16, 6)            // config 5: CD 2D p=6 (ws2: s / u^{k+1} bypass smem)
    IHDG_WS3(7, 3, 4, 2, 16, IHDG_WS3_NS)  // config 5: CD 2D p=6 (ws3: q in the consumers, DFMA norm warps)
    {2, 7, 3, 4, 2, 16, 147, launch_ws4_t<7, 3, 4, 2, IHDG_WS4_NS>, 0, 2},  // config 5 (ws4: two consumer teams)
    {2, 7, 3, 4, 2, 16, 147, launch_v3_t<2, 7, 3, 4, 2, IHDG_C5V3_NS, IHDG_C5V3_NCW, 2, IHDG_C5V3_NQW>, 1, 3},  // config 5 (v3)
    IHDG_WS(7, 3, 4, 2, 16, IHDG_WS5_NS)   // config 5: CD 2D p=6 (warp-specialised)
    IHDG_WS(5, 3, 4, 2, 16, 4)             // configs 2/3: CD / SW 2D p=4
    IHDG_STREAM(3, 4, 1, 3, 1, 32, 3, 4)   // config 4: transport 3D p=3
};

// Returns the entry usable for these args, or nullptr (generic kernel).
const StreamEntry* stream_entry(const ihdg_sweep_args* a) {
  static int forced_generic = -1;
  if (forced_generic < 0) {
    const char* s = std::getenv("IHDG_SWEEP_IMPL");
    forced_generic = (s != nullptr && std::strcmp(s, "generic") == 0) ? 1 : 0;
  }
  if (forced_generic) return nullptr;
  static int no_v3 = -1;
  if (no_v3 < 0) {
    const char* s = std::getenv("IHDG_SWEEP_IMPL");
    no_v3 = (s != nullptr && (std::strcmp(s, "ws") == 0 || std::strcmp(s, "stream") == 0)) ? 1 : 0;
  }
  // IHDG_SWEEP_IMPL: "ws2" opts in to the experimental ws2 kernel (slower than
  // ws on config 5); "ws"/"stream" skip v3; "generic" skips all
  static int want_ws2 = -1;
  if (want_ws2 < 0) {
    const char* s = std::getenv("IHDG_SWEEP_IMPL");
    want_ws2 = (s != nullptr && std::strcmp(s, "ws2") == 0) ? 1 : 0;
  }
  // "ws3" opts in to k_sweep_ws3 (slower than ws on config 5)
  static int want_ws4 = -1;
  if (want_ws4 < 0) {
    const char* s = std::getenv("IHDG_SWEEP_IMPL");
    want_ws4 = (s != nullptr && std::strcmp(s, "ws4") == 0) ? 1 : 0;
  }
  static int want_v3 = -1;
  if (want_v3 < 0) {
    const char* s = std::getenv("IHDG_SWEEP_IMPL");
    want_v3 = (s != nullptr && std::strcmp(s, "v3") == 0) ? 1 : 0;
  }
  static int want_ws3 = -1;
  if (want_ws3 < 0) {
    const char* s = std::getenv("IHDG_SWEEP_IMPL");
    want_ws3 = (s != nullptr && std::strcmp(s, "ws3") == 0) ? 1 : 0;
  }
  if (a->norm_kind != IHDG_NORM_VOLUME) return nullptr;
  if (a->scheme != IHDG_SCHEME_II) return nullptr;   // iHDG-I: generic kernel
  const ihdg_geom& g = a->g;
  int ncf = 0, maxw = 0;
  for (int f = 0; f < 2 * g.dim; ++f) {
    if (!a->coupled[f]) continue;
    ++ncf;
    int w = 0;
    for (int c = 0; c < g.ncomp; ++c) w += a->face_w[f][c] != 0.0;
    maxw = w > maxw ? w : maxw;
  }
  for (const StreamEntry& e : kStream) {
    if (e.D != g.dim || e.N1 != g.order + 1 || e.M != g.ncomp) continue;
    if (e.NCF != ncf || maxw > e.NWC) continue;
    if (e.v3 && no_v3) continue;
    if (e.ws3 == 1 && !want_ws3) continue;
    if (e.ws3 == 2 && !want_ws4) continue;
    if (e.ws3 == 3 && !want_v3) continue;
    if (e.launch == (int (*)(const ihdg_sweep_args*, cudaStream_t))launch_ws2_t<7, 3, 4, 2, 16, 6> && !want_ws2)
      continue;
    Geo geo;
    geo.init(g, e.E);
    if (geo.tile_len % e.E != 0) continue;                       // full tiles only
    if (g.cells[0] % (e.v3 ? 8 : e.E) != 0) continue;            // tiles inside one axis-0 row
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

// 1 if the streaming kernel is used for these args, 0 for the generic one.
int ihdg_stream_variant(const ihdg_sweep_args* a) { return ihdg::stream_entry(a) != nullptr ? 1 : 0; }

// Launch the streaming kernel if applicable. Returns 1 launched, 0 not
// applicable, <0 on launch error.
int ihdg_stream_launch(const ihdg_sweep_args* a, cudaStream_t st) {
  const ihdg::StreamEntry* e = ihdg::stream_entry(a);
  if (e == nullptr) return 0;
  int rc = e->launch(a, st);
  return rc == 0 ? 1 : rc;
}
