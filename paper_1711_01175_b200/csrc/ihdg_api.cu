// extern "C" entry points of libihdg_cuda.so (declared in include/ihdg.h).
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ihdg_kernels.cuh"
#include "ihdg_setup_kernels.cuh"

using namespace ihdg;

int ihdg_stream_launch(const ihdg_sweep_args* a, cudaStream_t st, cudaError_t* err);
const char* ihdg_stream_kernel_name(const ihdg_sweep_args* a);
int ihdg_stream_set_impl(const char* name);
int ihdg_stream_gram_kc(const ihdg_sweep_args* a);

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define IHDG_CUDA_TRY(expr)                                                                  \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) return set_err(IHDG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(IHDG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return IHDG_OK;
}

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

// SM count of the current device (cached per device ordinal)
int num_sms() {
  static int sms[64] = {0};
  const int dev = current_device() & 63;
  if (sms[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = n > 0 ? n : 148;
  }
  return sms[dev];
}

// ---- per-instantiation launchers -----------------------------------------
template <int D, int N1, int M>
int launch_sweep(const ihdg_sweep_args* a, cudaStream_t st) {
  using C = Cfg<D, N1, M>;
  static int grid_max_dev[64] = {0};   // per device ordinal
  int& grid_max = grid_max_dev[current_device() & 63];
  const size_t smem = SweepSmem<D, N1, M>::bytes;
  if (grid_max == 0) {
    IHDG_CUDA_TRY(cudaFuncSetAttribute(k_sweep<D, N1, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int nb = 0;
    IHDG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sweep<D, N1, M>, C::NT, smem));
    if (nb < 1) return set_err(IHDG_ERR_UNSUPPORTED, "sweep kernel does not fit on an SM");
    grid_max = nb * num_sms();
  }
  Geo geo;
  geo.init(a->g, C::TE);
  int64_t grid = geo.ntiles < grid_max ? geo.ntiles : grid_max;
  if (grid < 1) grid = 1;
  k_sweep<D, N1, M><<<(unsigned)grid, C::NT, smem, st>>>(*a);
  return check_launch("k_sweep");
}

template <int D, int N1, int M>
int launch_apply(const ihdg_class_apply_args* a, cudaStream_t st) {
  using C = Cfg<D, N1, M>;
  static int grid_max_dev[64] = {0};   // per device ordinal
  int& grid_max = grid_max_dev[current_device() & 63];
  const size_t smem = (size_t)C::NV * C::TE * sizeof(double);
  if (a->ncols > C::NV) return set_err(IHDG_ERR_ARG, "class_apply: ncols > NV");
  if (grid_max == 0) {
    IHDG_CUDA_TRY(cudaFuncSetAttribute(k_class_apply<D, N1, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int nb = 0;
    IHDG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_class_apply<D, N1, M>, C::NT, smem));
    if (nb < 1) nb = 1;
    grid_max = nb * num_sms();
  }
  Geo geo;
  geo.init(a->g, C::TE);
  int64_t grid = geo.ntiles < grid_max ? geo.ntiles : grid_max;
  if (grid < 1) return IHDG_OK;
  k_class_apply<D, N1, M><<<(unsigned)grid, C::NT, smem, st>>>(*a);
  return check_launch("k_class_apply");
}

template <int D, int N1, int M>
int tile_elems() {
  return Cfg<D, N1, M>::TE;
}

struct Entry {
  int D, N1, M;
  int (*sweep)(const ihdg_sweep_args*, cudaStream_t);
  int (*apply)(const ihdg_class_apply_args*, cudaStream_t);
  int (*te)();
};

#define IHDG_ENTRY(D, N1, M) {D, N1, M, launch_sweep<D, N1, M>, launch_apply<D, N1, M>, tile_elems<D, N1, M>},

// Instantiated (dim, p+1, m): transport m=1; CD m=d+1; shallow water m=3 (2D).
const Entry kEntries[] = {
    IHDG_ENTRY(1, 2, 1) IHDG_ENTRY(1, 3, 1) IHDG_ENTRY(1, 4, 1) IHDG_ENTRY(1, 5, 1) IHDG_ENTRY(1, 6, 1)
    IHDG_ENTRY(1, 7, 1)
    IHDG_ENTRY(1, 2, 2) IHDG_ENTRY(1, 3, 2) IHDG_ENTRY(1, 4, 2) IHDG_ENTRY(1, 5, 2)
    IHDG_ENTRY(2, 2, 1) IHDG_ENTRY(2, 3, 1) IHDG_ENTRY(2, 4, 1) IHDG_ENTRY(2, 5, 1) IHDG_ENTRY(2, 6, 1)
    IHDG_ENTRY(2, 7, 1)
    IHDG_ENTRY(2, 2, 3) IHDG_ENTRY(2, 3, 3) IHDG_ENTRY(2, 4, 3) IHDG_ENTRY(2, 5, 3) IHDG_ENTRY(2, 6, 3)
    IHDG_ENTRY(2, 7, 3)
    IHDG_ENTRY(3, 2, 1) IHDG_ENTRY(3, 3, 1) IHDG_ENTRY(3, 4, 1) IHDG_ENTRY(3, 5, 1)
    IHDG_ENTRY(3, 2, 4) IHDG_ENTRY(3, 3, 4) IHDG_ENTRY(3, 4, 4) IHDG_ENTRY(3, 5, 4)
};

const Entry* find_entry(int D, int order, int M) {
  for (const Entry& e : kEntries)
    if (e.D == D && e.N1 == order + 1 && e.M == M) return &e;
  return nullptr;
}

int check_geom(const ihdg_geom& g) {
  if (g.dim < 1 || g.dim > 3) return set_err(IHDG_ERR_ARG, "dim must be 1, 2 or 3");
  if (g.order < 1 || g.order > 10) return set_err(IHDG_ERR_ARG, "order must be in 1..10");
  if (g.ncomp < 1 || g.ncomp > IHDG_MAX_COMP) return set_err(IHDG_ERR_ARG, "ncomp must be in 1..4");
  for (int a = 0; a < g.dim; ++a)
    if (g.cells[a] < 1) return set_err(IHDG_ERR_ARG, "cell counts must be positive");
  if (g.layer_begin < 0 || g.layer_end > g.cells[g.dim - 1] || g.layer_end <= g.layer_begin)
    return set_err(IHDG_ERR_ARG, "bad layer range");
  return IHDG_OK;
}

int64_t layer_size(const ihdg_geom& g) {
  int64_t ls = 1;
  for (int a = 0; a < g.dim - 1; ++a) ls *= g.cells[a];
  return ls;
}

}  // namespace

extern "C" {

int ihdg_abi_version(void) { return IHDG_ABI_VERSION; }

const char* ihdg_last_error(void) { return g_err.c_str(); }

int64_t ihdg_struct_size(int32_t which) {
  switch (which) {
    case 0: return sizeof(ihdg_geom);
    case 1: return sizeof(ihdg_iter_state);
    case 2: return sizeof(ihdg_assembly_args);
    case 3: return sizeof(ihdg_class_apply_args);
    case 4: return sizeof(ihdg_field_args);
    case 5: return sizeof(ihdg_quad_args);
    case 6: return sizeof(ihdg_sweep_args);
    case 7: return sizeof(ihdg_finalize_args);
    case 8: return sizeof(ihdg_trace_args);
    case 9: return sizeof(ihdg_error_args);
    case 10: return sizeof(ihdg_elem_error_args);
    case 11: return sizeof(ihdg_face_energy_args);
    case 12: return sizeof(ihdg_halo_args);
    default: return -1;
  }
}

int ihdg_supported(int32_t dim, int32_t order, int32_t ncomp) {
  return find_entry(dim, order, ncomp) != nullptr ? 1 : 0;
}

int32_t ihdg_tile_elems(int32_t dim, int32_t order, int32_t ncomp) {
  const Entry* e = find_entry(dim, order, ncomp);
  return e ? e->te() : -1;
}

int64_t ihdg_tile_count(const ihdg_geom* g) {
  if (g == nullptr || check_geom(*g) != IHDG_OK) return -1;
  const Entry* e = find_entry(g->dim, g->order, g->ncomp);
  if (e == nullptr) return -1;
  Geo geo;
  geo.init(*g, e->te());
  return geo.ntiles;
}

int ihdg_assemble(const ihdg_assembly_args* a, void* stream) {
  if (a == nullptr) return set_err(IHDG_ERR_ARG, "null args");
  if (a->dim < 1 || a->dim > 3 || a->order < 1 || a->ncomp < 1 || a->n_class < 1)
    return set_err(IHDG_ERR_ARG, "bad assembly dims");
  cudaStream_t st = (cudaStream_t)stream;
  AsmDims dm;
  dm.D = a->dim;
  dm.N1 = a->order + 1;
  dm.NP = 1;
  for (int i = 0; i < dm.D; ++i) dm.NP *= dm.N1;
  dm.NF = dm.NP / dm.N1;
  dm.NV = a->ncomp * dm.NP;
  dm.KIN = 2 * dm.D * dm.NF * (a->kin_blocks > 1 ? a->kin_blocks : 1);
  dm.nr = a->nr;
  int* perm = nullptr;
  IHDG_CUDA_TRY(cudaMallocAsync((void**)&perm, sizeof(int) * dm.NV * a->n_class, st));
  k_assemble_build<<<a->n_class, 256, 0, st>>>(*a, dm);
  int rc = check_launch("k_assemble_build");
  if (rc) return rc;
  k_gauss_jordan<<<a->n_class, 512, 2 * dm.NV * sizeof(double), st>>>(*a, dm, perm);
  rc = check_launch("k_gauss_jordan");
  if (rc) return rc;
  k_assemble_lift<<<a->n_class, 256, 0, st>>>(*a, dm);
  rc = check_launch("k_assemble_lift");
  if (rc) return rc;
  IHDG_CUDA_TRY(cudaFreeAsync(perm, st));
  return IHDG_OK;
}

int ihdg_class_apply(const ihdg_class_apply_args* a, void* stream) {
  if (a == nullptr) return set_err(IHDG_ERR_ARG, "null args");
  int rc = check_geom(a->g);
  if (rc) return rc;
  const Entry* e = find_entry(a->g.dim, a->g.order, a->g.ncomp);
  if (e == nullptr) return set_err(IHDG_ERR_UNSUPPORTED, "no kernel instantiated for this (dim, order, ncomp)");
  return e->apply(a, (cudaStream_t)stream);
}

int ihdg_eval_field(const ihdg_field_args* a, void* stream) {
  if (a == nullptr) return set_err(IHDG_ERR_ARG, "null args");
  int rc = check_geom(a->g);
  if (rc) return rc;
  Geo geo;
  geo.init(a->g, 1);
  int64_t npts = 1;
  for (int i = 0; i < a->g.dim; ++i) npts *= a->npts1d;
  int64_t total = geo.nloc * npts;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 8 * num_sms() * 8) blocks = 8 * num_sms() * 8;
  if (blocks < 1) return IHDG_OK;
  k_eval_field<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(*a);
  return check_launch("k_eval_field");
}

int ihdg_quad_project(const ihdg_quad_args* a, void* stream) {
  if (a == nullptr) return set_err(IHDG_ERR_ARG, "null args");
  int rc = check_geom(a->g);
  if (rc) return rc;
  Geo geo;
  geo.init(a->g, 1);
  int64_t np = 1;
  for (int i = 0; i < a->g.dim; ++i) np *= (a->g.order + 1);
  int64_t total = geo.nloc * np;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 64 * num_sms()) blocks = 64 * num_sms();
  if (blocks < 1) return IHDG_OK;
  k_quad_project<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(*a);
  return check_launch("k_quad_project");
}

static int do_sweep(const Entry* e, const ihdg_sweep_args* a, cudaStream_t st) {
  cudaError_t ce = cudaSuccess;
  const int rc = ihdg_stream_launch(a, st, &ce);
  if (rc == 1) return IHDG_OK;
  if (rc < 0)
    return set_err(IHDG_ERR_CUDA, std::string(ihdg_stream_kernel_name(a)) + " launch: " + cudaGetErrorString(ce));
  return e->sweep(a, st);
}

int ihdg_sweep(const ihdg_sweep_args* a, void* stream) {
  if (a == nullptr) return set_err(IHDG_ERR_ARG, "null args");
  int rc = check_geom(a->g);
  if (rc) return rc;
  const Entry* e = find_entry(a->g.dim, a->g.order, a->g.ncomp);
  if (e == nullptr) return set_err(IHDG_ERR_UNSUPPORTED, "no kernel instantiated for this (dim, order, ncomp)");
  return do_sweep(e, a, (cudaStream_t)stream);
}

const char* ihdg_sweep_kernel(const ihdg_sweep_args* a) {
  if (a == nullptr || check_geom(a->g) != IHDG_OK) return nullptr;
  if (find_entry(a->g.dim, a->g.order, a->g.ncomp) == nullptr) return nullptr;
  const char* s = ihdg_stream_kernel_name(a);
  return s != nullptr ? s : "k_sweep";
}

int ihdg_sweep_gram_kc(const ihdg_sweep_args* a) {
  if (a == nullptr || check_geom(a->g) != IHDG_OK) return 0;
  return ihdg_stream_gram_kc(a);
}

int ihdg_set_sweep_impl(const char* name) {
  if (ihdg_stream_set_impl(name) != 0)
    return set_err(IHDG_ERR_ARG, std::string("unknown sweep impl '") + (name ? name : "(null)") +
                                     "' (auto, v3, v5, ws, stream, generic)");
  return IHDG_OK;
}

int ihdg_finalize(const ihdg_finalize_args* a, void* stream) {
  if (a == nullptr) return set_err(IHDG_ERR_ARG, "null args");
  k_finalize<<<1, 256, 0, (cudaStream_t)stream>>>(*a);
  return check_launch("k_finalize");
}

int ihdg_layer_sums(const double* tile_partials, int64_t n_rows, int64_t row_len, double* out, void* stream) {
  if (tile_partials == nullptr || out == nullptr || n_rows < 0 || row_len < 1) return set_err(IHDG_ERR_ARG, "bad args");
  if (n_rows == 0) return IHDG_OK;
  int64_t grid = (n_rows + 3) / 4;   // 4 warps (rows) per CTA
  if (grid > 8 * num_sms()) grid = 8 * num_sms();
  k_layer_sums<<<(unsigned)grid, 128, 0, (cudaStream_t)stream>>>(tile_partials, n_rows, row_len, out);
  return check_launch("k_layer_sums");
}

static int halo_copy(const ihdg_halo_args* a, int unpack, cudaStream_t st) {
  if (a == nullptr || a->buf == nullptr || a->packed == nullptr || a->idx == nullptr || a->n_idx < 1)
    return set_err(IHDG_ERR_ARG, "null / empty halo args");
  int rc = check_geom(a->g);
  if (rc) return rc;
  if (a->layer < 0 || a->layer > 3 || (unpack ? (a->layer == 1 || a->layer == 2) : (a->layer == 0 || a->layer == 3)))
    return set_err(IHDG_ERR_ARG, "halo layer: pack reads layer 1/2, unpack writes layer 0/3");
  const int64_t total = layer_size(a->g) * a->n_idx;
  int64_t grid = (total + 255) / 256;
  if (grid > 4 * num_sms()) grid = 4 * num_sms();
  k_halo_copy<<<(unsigned)grid, 256, 0, st>>>(*a, unpack);
  return check_launch("k_halo_copy");
}

int ihdg_halo_pack(const ihdg_halo_args* a, void* stream) { return halo_copy(a, 0, (cudaStream_t)stream); }
int ihdg_halo_unpack(const ihdg_halo_args* a, void* stream) { return halo_copy(a, 1, (cudaStream_t)stream); }

int ihdg_extract_trace(const ihdg_trace_args* a, void* stream) {
  if (a == nullptr) return set_err(IHDG_ERR_ARG, "null args");
  int rc = check_geom(a->g);
  if (rc) return rc;
  if (a->g.layer_begin != 0 || a->g.layer_end != a->g.cells[a->g.dim - 1])
    return set_err(IHDG_ERR_UNSUPPORTED, "trace extraction needs the whole mesh on one rank");
  k_extract_trace<<<4 * num_sms(), 256, 0, (cudaStream_t)stream>>>(*a);
  return check_launch("k_extract_trace");
}

int ihdg_copy_state(const ihdg_geom* g, const double* src, double* dst, void* stream) {
  if (g == nullptr) return set_err(IHDG_ERR_ARG, "null args");
  int rc = check_geom(*g);
  if (rc) return rc;
  int64_t np = 1;
  for (int i = 0; i < g->dim; ++i) np *= (g->order + 1);
  const int64_t ls = layer_size(*g);
  const int64_t n = ((g->layer_end - g->layer_begin) * ls + 2 * ls) * g->ncomp * np;
  IHDG_CUDA_TRY(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return IHDG_OK;
}

// A batch of sweeps as one CUDA graph (launch-bound small meshes): captured
// once per (args, buffers, batch, stream) and replayed; an even batch keeps
// the buffer parity of every replay at buf0 -> buf1.
struct SweepGraph {
  ihdg_sweep_args a;
  ihdg_error_args e;
  bool has_e = false;
  double* b0 = nullptr;
  double* b1 = nullptr;
  int nb = 0;
  cudaStream_t st = nullptr;
  cudaGraphExec_t exec = nullptr;
};

// CUDA-graph replay of sweep batches: on unless IHDG_NO_GRAPH is set, and
// switchable at run time (ihdg_set_graphs)
static std::atomic<int> g_graphs{-1};

static bool graphs_enabled() {
  int on = g_graphs.load();
  if (on < 0) {
    const char* s = std::getenv("IHDG_NO_GRAPH");
    int expect = -1;
    g_graphs.compare_exchange_strong(expect, (s != nullptr && s[0] != '\0' && s[0] != '0') ? 0 : 1);
    on = g_graphs.load();
  }
  return on == 1;
}

extern "C" int ihdg_set_graphs(int on) {
  g_graphs.store(on ? 1 : 0);
  return IHDG_OK;
}

static int do_error(const ihdg_error_args* e, cudaStream_t st);

static cudaGraphExec_t sweep_graph(const Entry* e, const ihdg_sweep_args& a, const ihdg_error_args* ea, double* b0,
                                   double* b1, int nb, cudaStream_t st) {
  static thread_local SweepGraph cache_dev[8];   // per device ordinal (mod 8)
  SweepGraph& cache = cache_dev[current_device() & 7];
  const bool has_e = ea != nullptr;
  if (cache.exec != nullptr && cache.b0 == b0 && cache.b1 == b1 && cache.nb == nb && cache.st == st &&
      std::memcmp(&cache.a, &a, sizeof(a)) == 0 && cache.has_e == has_e &&
      (!has_e || std::memcmp(&cache.e, ea, sizeof(*ea)) == 0))
    return cache.exec;
  if (cache.exec != nullptr) {
    cudaGraphExecDestroy(cache.exec);
    cache.exec = nullptr;
  }
  if (cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  ihdg_sweep_args s = a;
  bool ok = true;
  for (int j = 0; j < nb && ok; ++j) {
    s.u_old = (j & 1) ? b1 : b0;
    s.u_new = (j & 1) ? b0 : b1;
    ok = do_sweep(e, &s, st) == IHDG_OK;
    if (ok && has_e) {
      ihdg_error_args x = *ea;
      x.u = s.u_new;
      ok = do_error(&x, st) == IHDG_OK;
    }
  }
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(st, &g);
  cudaGraphExec_t ex = nullptr;
  if (ok && ce == cudaSuccess && g != nullptr && cudaGraphInstantiate(&ex, g, 0) == cudaSuccess) {
    cache.a = a;
    if (has_e) cache.e = *ea;
    cache.has_e = has_e;
    cache.b0 = b0;
    cache.b1 = b1;
    cache.nb = nb;
    cache.st = st;
    cache.exec = ex;
  } else {
    ex = nullptr;
  }
  if (g != nullptr) cudaGraphDestroy(g);
  cudaGetLastError();
  return ex;
}

static int64_t error_tiles(const ihdg_geom& g) {
  Geo geo;
  geo.init(g, ERR_TE);
  return geo.ntiles;
}

static int do_error(const ihdg_error_args* e, cudaStream_t st) {
  const int64_t nt = error_tiles(e->g);
  int64_t grid = nt < 4 * num_sms() ? nt : 4 * num_sms();
  if (grid < 1) grid = 1;
  k_error_norm<<<(unsigned)grid, 256, 0, st>>>(*e);
  return check_launch("k_error_norm");
}

int ihdg_error_norm(const ihdg_error_args* e, void* stream) {
  if (e == nullptr || e->u == nullptr || e->ue_q == nullptr || e->state == nullptr)
    return set_err(IHDG_ERR_ARG, "null args");
  int rc = check_geom(e->g);
  if (rc) return rc;
  if (e->nq < 1 || e->nq > 16 || e->g.order + 1 > 8) return set_err(IHDG_ERR_ARG, "nq / order out of range");
  if (e->mode < 0 || e->mode > 2) return set_err(IHDG_ERR_ARG, "mode must be 0, 1 or 2");
  if (e->mode != 0 && e->succ_partials == nullptr) return set_err(IHDG_ERR_ARG, "modes 1/2 need the sweep partials");
  return do_error(e, (cudaStream_t)stream);
}

int64_t ihdg_error_tile_count(const ihdg_geom* g) { return g == nullptr ? -1 : error_tiles(*g); }

int ihdg_elem_error(const ihdg_elem_error_args* a, void* stream) {
  if (a == nullptr || a->u == nullptr || a->r == nullptr || a->chol1d == nullptr || a->err2 == nullptr)
    return set_err(IHDG_ERR_ARG, "null args");
  int rc = check_geom(a->g);
  if (rc) return rc;
  if (a->g.order + 1 > 8) return set_err(IHDG_ERR_ARG, "order out of range (p <= 7)");
  Geo geo;
  geo.init(a->g, 1);
  if (geo.nloc == 0) return IHDG_OK;
  const int64_t grid = geo.nloc < 8 * num_sms() ? geo.nloc : 8 * num_sms();
  k_elem_error<<<(unsigned)grid, 128, 0, (cudaStream_t)stream>>>(*a);
  rc = check_launch("k_elem_error");
  if (rc || a->total == nullptr) return rc;
  k_fixed_total<<<1, 256, 0, (cudaStream_t)stream>>>(a->err2, geo.nloc, a->total);
  return check_launch("k_fixed_total");
}

int ihdg_face_energy(const ihdg_face_energy_args* a, void* stream) {
  if (a == nullptr || a->t == nullptr || a->chol1d == nullptr || a->e2 == nullptr)
    return set_err(IHDG_ERR_ARG, "null args");
  int rc = check_geom(a->g);
  if (rc) return rc;
  if (a->g.order + 1 > 8) return set_err(IHDG_ERR_ARG, "order out of range (p <= 7)");
  Geo geo;
  geo.init(a->g, 1);
  if (geo.lb != 0 || geo.le != geo.c[geo.D - 1]) return set_err(IHDG_ERR_ARG, "face energy needs the whole mesh");
  int64_t nfaces = 0;
  for (int ax = 0; ax < geo.D; ++ax) {
    int64_t ntan = 1;
    for (int b = 0; b < geo.D; ++b)
      if (b != ax) ntan *= geo.c[b];
    nfaces += (geo.c[ax] + (geo.per[ax] ? 0 : 1)) * ntan;
  }
  int64_t grid = (nfaces + 127) / 128;
  if (grid > 8 * num_sms()) grid = 8 * num_sms();
  if (grid < 1) grid = 1;
  k_face_energy<<<(unsigned)grid, 128, 0, (cudaStream_t)stream>>>(*a);
  rc = check_launch("k_face_energy");
  if (rc || a->total == nullptr) return rc;
  k_fixed_total<<<1, 256, 0, (cudaStream_t)stream>>>(a->e2, nfaces, a->total);
  return check_launch("k_fixed_total");
}

static int iterate_impl(const ihdg_sweep_args* a0, const ihdg_error_args* e0, double* buf0, double* buf1,
                        int32_t batch, void* stream, ihdg_iter_state* state_out, int64_t* n_launched);

int ihdg_iterate(const ihdg_sweep_args* a0, double* buf0, double* buf1, int32_t batch, void* stream,
                 ihdg_iter_state* state_out, int64_t* n_launched) {
  return iterate_impl(a0, nullptr, buf0, buf1, batch, stream, state_out, n_launched);
}

int ihdg_iterate_exact(const ihdg_sweep_args* a0, const ihdg_error_args* e0, double* buf0, double* buf1,
                       int32_t batch, void* stream, ihdg_iter_state* state_out, int64_t* n_launched) {
  if (e0 == nullptr) return set_err(IHDG_ERR_ARG, "null error args");
  return iterate_impl(a0, e0, buf0, buf1, batch, stream, state_out, n_launched);
}

static int iterate_impl(const ihdg_sweep_args* a0, const ihdg_error_args* e0, double* buf0, double* buf1,
                        int32_t batch, void* stream, ihdg_iter_state* state_out, int64_t* n_launched) {
  if (a0 == nullptr || buf0 == nullptr || buf1 == nullptr || state_out == nullptr)
    return set_err(IHDG_ERR_ARG, "null args");
  if (batch < 1) batch = 1;
  int rc = check_geom(a0->g);
  if (rc) return rc;
  const Entry* e = find_entry(a0->g.dim, a0->g.order, a0->g.ncomp);
  if (e == nullptr) return set_err(IHDG_ERR_UNSUPPORTED, "no kernel instantiated for this (dim, order, ncomp)");
  static thread_local ihdg_iter_state* hs = nullptr;
  if (hs == nullptr) IHDG_CUDA_TRY(cudaMallocHost((void**)&hs, sizeof(ihdg_iter_state)));
  cudaStream_t st = (cudaStream_t)stream;
  if (graphs_enabled() && (st == nullptr || st == cudaStreamLegacy || st == cudaStreamPerThread)) {
    // the default stream cannot be captured: run the loop on a private
    // stream (per device) ordered after the caller's work (the call is synchronous)
    static thread_local cudaStream_t own_dev[8] = {nullptr};
    static thread_local cudaEvent_t ev_dev[8] = {nullptr};
    const int slot = current_device() & 7;
    cudaStream_t& own = own_dev[slot];
    cudaEvent_t& ev = ev_dev[slot];
    if (own == nullptr) {
      IHDG_CUDA_TRY(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
      IHDG_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    IHDG_CUDA_TRY(cudaEventRecord(ev, st));
    IHDG_CUDA_TRY(cudaStreamWaitEvent(own, ev, 0));
    st = own;
  }
  ihdg_sweep_args a = *a0;
  a.finalize = e0 == nullptr ? 1 : 0;   // exact rule: K5 finalizes
  a.u_old = a.u_new = nullptr;
  ihdg_error_args ex{};
  if (e0 != nullptr) {
    ex = *e0;
    ex.mode = e0->mode == 2 ? 2 : 1;   // 2: vs-direct rule, else the exact-solution rule
    ex.u = nullptr;
    ex.succ_partials = a.tile_partials;
    ex.state = a.state;
  }
  const ihdg_error_args* ep = e0 != nullptr ? &ex : nullptr;
  int64_t launched = 0;
  int32_t seen_iters = -1;
  // sweeps after the stop are no-ops on the device, so a batch rounded up to
  // an even count changes nothing but the launch count
  const int nb = batch + (batch & 1);
  cudaGraphExec_t gx = graphs_enabled() ? sweep_graph(e, a, ep, buf0, buf1, nb, st) : nullptr;
  for (;;) {
    if (gx != nullptr) {
      IHDG_CUDA_TRY(cudaGraphLaunch(gx, st));
      launched += nb;
    } else {
      for (int j = 0; j < batch; ++j) {
        a.u_old = (launched & 1) ? buf1 : buf0;
        a.u_new = (launched & 1) ? buf0 : buf1;
        rc = do_sweep(e, &a, st);
        if (rc) return rc;
        if (ep != nullptr) {
          ex.u = a.u_new;
          rc = do_error(&ex, st);
          if (rc) return rc;
        }
        ++launched;
      }
    }
    IHDG_CUDA_TRY(cudaMemcpyAsync(hs, a0->state, sizeof(ihdg_iter_state), cudaMemcpyDeviceToHost, st));
    IHDG_CUDA_TRY(cudaStreamSynchronize(st));
    if (hs->status != IHDG_RUNNING) break;
    // a batch of live sweeps always advances the count (every sweep either
    // finalizes or the status leaves RUNNING): no progress means the kernels
    // did not run, so fail instead of polling forever
    if (hs->iters <= seen_iters || hs->iters > hs->max_iters)
      return set_err(IHDG_ERR_CUDA, "ihdg_iterate: the device iteration count stopped advancing (" +
                                        std::to_string(hs->iters) + " after " + std::to_string(launched) +
                                        " launched sweeps)");
    seen_iters = hs->iters;
  }
  *state_out = *hs;
  if (n_launched) *n_launched = launched;
  return IHDG_OK;
}

}  // extern "C"
