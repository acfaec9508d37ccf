/*
 * ihdg.h -- C ABI of libihdg_cuda.so, the B200 (sm_100a) implementation of
 * the iHDG-II element sweep (arXiv 1711.01175, Algorithm 1).
 *
 * Which reference interface this replaces
 * ---------------------------------------
 * The reference package routes every iteration of `ihdg.iteration.run`
 * through a native element map, the Cython/OpenMP module
 * `ihdg._kernels._sweep_cy` (pkg/setup.py:13-19).  Its source is absent from
 * the reference, so the seam is defined by its callers:
 *
 *   ihdg_assemble      <- local_solvers.assemble_transport / _shallow_water /
 *                         _convection_diffusion + "factor once"
 *
 *   ihdg_class_apply   <- the RHS builder of LocalSystem:
 *                         s = A^-1 b  (forcing) and s = P u^m (time level)
 *                         for run_time_dependent
 *   ihdg_sweep         <- one pass of the parallel map
 *                         `parallel-for K: apply_local(...)` (SPEC.md:276-284,
 *                         297-298) + the stopping norm l2_norm of the
 *                         successive difference (
 *                         PAPER.md:1308-1311) + divergence detector
 *   ihdg_finalize      <- the post-barrier stopping check when the
 *                         tile partials were gathered from several ranks
 *   ihdg_iterate       <- the whole `while not converged` loop of Algorithm 1
 *                          on one device
 *   ihdg_eval_field    <- basis.project (nodal interpolation)
 *                         and forcing evaluation at quadrature points, for the
 *                         seeded Fourier / Gaussian fields of BASELINE.json
 *   ihdg_quad_project  <- (f, v)_K of the RHS builder
 *   ihdg_extract_trace <- the single-valued trace returned by run/solve_direct
 *                         (SURVEY.md Appendix B.8), face order of
 *                         mesh.py:89-125
 *
 * Conventions
 * -----------
 *  - Every pointer argument named in an args struct is a DEVICE pointer unless
 *    the field comment says "host".  No pointer is retained after a call.
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *  - Return value: IHDG_OK (0) or a negative IHDG_ERR_*; ihdg_last_error()
 *    returns a thread-local message for the last failure.
 *  - FieldState layout: element-major (Nel, m, (p+1)^d)
 *    fp64, nodes lexicographic with axis 0 fastest (mesh.py:155-164).
 *    "Ghost-padded" buffers carry one extra layer of elements (the slowest
 *    axis, dim-1) before and after the local range for the halo exchange of
 *    a strip partition; the local FieldState is the contiguous middle slice.
 */
#ifndef IHDG_H
#define IHDG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IHDG_ABI_VERSION 3
#define IHDG_MAX_DIM 3
#define IHDG_MAX_COMP 4
#define IHDG_MAX_FACE 6
#define IHDG_CHOL_MAX 64 /* (order+1)^2 entries of the 1D mass Cholesky factor, order <= 7 */

/* return codes */
#define IHDG_OK 0
#define IHDG_ERR_ARG (-1)
#define IHDG_ERR_CUDA (-2)
#define IHDG_ERR_UNSUPPORTED (-3)
#define IHDG_ERR_SINGULAR (-4)

/* iteration status (SPEC.md:321 status in {converged, diverged, max-iter}) */
#define IHDG_RUNNING 0
#define IHDG_CONVERGED 1
#define IHDG_DIVERGED 2
#define IHDG_NAN 3
#define IHDG_MAXITER 4

/* stopping norms */
#define IHDG_NORM_VOLUME 0 /* ||u^k - u^{k-1}||_{L2(Omega)} */
#define IHDG_SCHEME_II 0   /* iHDG-II: own iterate k+1 in the trace */
#define IHDG_SCHEME_I 1    /* iHDG-I: all-iterate-k trace */
#define IHDG_NORM_TRACE 1  /* skeleton L2 norm of the trace update */

/* Structured-mesh geometry of one rank's strip (mesh.py:33-77).  Elements are
 * lexicographic, axis 0 fastest; the strip is the element layers
 * [layer_begin, layer_end) of the slowest axis (dim-1). */
typedef struct {
  int32_t dim;          /* 1, 2 or 3 */
  int32_t order;        /* p, 1..10 (kernels instantiated for a subset) */
  int32_t ncomp;        /* m: 1 transport, d+1 CD, 3 shallow water */
  int32_t pad0;
  int64_t cells[3];     /* global cells per axis */
  int32_t periodic[3];  /* per-axis periodic flag */
  int32_t pad1;
  int64_t layer_begin;  /* local range along axis dim-1 */
  int64_t layer_end;
} ihdg_geom;

/* Device-resident control block of one iteration (Algorithm 1 loop). */
typedef struct {
  int32_t status;       /* IHDG_RUNNING / CONVERGED / ... */
  int32_t iters;        /* sweeps executed (SPEC.md:391 counting rule) */
  int32_t max_iters;
  uint32_t ticket;      /* last-block election counter, must start at 0 */
  double tol;           /* default 1e-10 */
  double first_norm;
  double last_norm;
  double diverge_factor;/* 1e6 */
  double last_err;      /* exact-solution rule: ||u^k - u^e||_{L2} of the latest iterate */
} ihdg_iter_state;

/* K1: assemble A (and the neighbour-coupling B, time-level R) per operator
 * class from a Kronecker term list, invert A by Gauss-Jordan with partial
 * pivoting, and form L = A^-1 B and P = A^-1 R.
 * A term adds coef * (op[0] (x) op[1] (x) op[2]) (axis 0 fastest) into one
 * (row component, column block) block of one target of one class.
 * Targets: 0 = A (col block = component), 1 = B (col block = local face
 * 2*axis+side, columns = face nodes), 2 = R (col block = time component). */
typedef struct {
  int32_t dim, order, ncomp, n_class;
  int32_t n_ops;
  int32_t n_terms;
  int32_t nr;              /* R columns (n_time_comp * (p+1)^d), may be 0 */
  int32_t kin_blocks;      /* B column blocks per face (face nodes each): 0/1 = one neighbour
                              scalar, 2 = raw neighbour values of 2 components (per-element
                              operators), 4 = + the element's own 2 (iHDG-I) */
  const double* ops1d;     /* [n_ops][N1][N1] row-major (device) */
  const int32_t* op_ncols; /* [n_ops], N1 or 1 (column vector) (device) */
  const int32_t* terms;    /* [n_terms][8] = class,target,row_comp,col_block,op0,op1,op2,unused (device) */
  const double* coefs;     /* [n_terms] (device) */
  double* A;               /* out [n_class][NV][NV] */
  double* Ainv;            /* out [n_class][NV][NV] */
  double* AinvT;           /* out [n_class][NV][NV], AinvT[c][j][i] = Ainv[c][i][j] */
  double* B;               /* workspace [n_class][NV][KIN] */
  double* R;               /* workspace [n_class][NV][nr] (may be NULL if nr == 0) */
  double* LT;              /* out [n_class][KIN][NV] = (A^-1 B)^T */
  double* PT;              /* out [n_class][nr][NV] = (A^-1 R)^T (may be NULL) */
  double* min_pivot;       /* out [n_class] min |pivot| of the factorization */
} ihdg_assembly_args;

/* K4: per-element class operator application
 *   out[e][r] (+)= sum_k opT[class(e)][k][r] * in[e][in_offset + k]        */
typedef struct {
  ihdg_geom g;
  const double* opT;          /* [n_class][ncols][NV] */
  const int32_t* class_of_mask; /* [64] boundary-face mask -> class */
  const double* in;           /* element stride in_stride doubles */
  double* out;                /* element stride NV doubles */
  int64_t in_stride;
  int32_t in_offset;
  int32_t ncols;
  int32_t in_ghost;           /* in is ghost-padded */
  int32_t out_ghost;          /* out is ghost-padded */
  int32_t accumulate;         /* out += ... instead of out = ... */
  int32_t per_element;        /* 1: operator class = local element index (per-element operators) */
} ihdg_class_apply_args;

/* Analytic fields evaluated at the tensor points of every local element:
 * kind 0: sum_j a_j sin(2 pi k_j . x + phi_j), params [nmodes][2+dim] = a, k.., phi
 * kind 1: a exp(-|x-c|^2 / (2 w^2)),          params [nmodes][2+dim] = a, c.., w (summed) */
typedef struct {
  ihdg_geom g;
  double lo[3];
  double h[3];
  const double* ref1d;   /* [npts1d] reference points on [-1,1] (device) */
  const double* params;  /* (device) */
  double* out;
  int64_t out_stride;    /* element stride in doubles */
  int32_t out_offset;
  int32_t out_ghost;
  int32_t npts1d;
  int32_t kind;
  int32_t nmodes;
  int32_t pad0;
} ihdg_field_args;

/* b[e][out_offset + i] = jac * sum_q prod_a Bq[i_a][q_a] * fq[e][q]          */
typedef struct {
  ihdg_geom g;
  const double* Bq;      /* [N1][nq] = V^T diag(w) (device) */
  const double* fq;      /* [Nel_local][nq^d] */
  double* out;
  int64_t out_stride;
  int32_t out_offset;
  int32_t nq;
  double jac;
} ihdg_quad_args;

/* K2+K3: one fused iHDG-II sweep over the local strip:
 *   q[K][f][n] = sum_c face_w[f][c] * u_old[nbr(K,f)][c][opposite face node n]
 *   u_new[K]   = s[K] + L[class(K)] q[K]                         (lifted local solve)
 *   partial    = sum_K ||u_new[K] - u_old[K]||^2                 (stopping norm)
 * With finalize = 1 the last CTA reduces the tile partials in a fixed order,
 * updates *state and turns all later sweeps into no-ops once converged. */
typedef struct {
  ihdg_geom g;
  const double* u_old;        /* ghost-padded */
  double* u_new;              /* ghost-padded */
  const double* s;            /* [Nel_local][NV] */
  const double* LT;           /* [n_class][KIN][NV] */
  const int32_t* class_of_mask; /* [64] */
  const double* chol1d;       /* [N1][N1] lower Cholesky factor C of the 1D reference mass, M1 = C C^T */
  double* tile_partials;      /* [n_tiles_local] */
  ihdg_iter_state* state;
  double* norm_hist;          /* [max_iters] or NULL */
  double face_w[IHDG_MAX_FACE][IHDG_MAX_COMP];
  double comp_w[IHDG_MAX_COMP];
  double out_w[IHDG_MAX_FACE][IHDG_MAX_COMP];
  double jac;                 /* volume Jacobian prod h_a/2 */
  double jac_face[IHDG_MAX_DIM]; /* face Jacobian of faces normal to axis a */
  int32_t coupled[IHDG_MAX_FACE];  /* face receives neighbour data */
  int32_t out_face[IHDG_MAX_FACE]; /* face contributes to the trace norm */
  int32_t norm_kind;          /* IHDG_NORM_VOLUME / IHDG_NORM_TRACE */
  int32_t finalize;           /* 1: fused last-CTA finalize (single rank) */
  int64_t tile_offset;        /* global index of this strip's first tile */
  double chol[IHDG_CHOL_MAX]; /* chol1d by value, row-major [N1][N1] (kernel-parameter
                                 constants for the DFMA stopping norm) */
  double own_w[IHDG_MAX_FACE][IHDG_MAX_COMP]; /* iHDG-I: q[K][f][n] += sum_c own_w[f][c] *
                                 u_old[K][c][face f node n] on every face, boundary or not
                                 (all-iterate-k trace); zero for iHDG-II */
  int32_t scheme;             /* IHDG_SCHEME_II / IHDG_SCHEME_I */
  int32_t pad1;
  /* Gram-form stopping norm (k_sweep_ws only; both NULL = the direct norm).
   * Within one solve, u^k = s + L q^{k-1} for k >= 1, so the successive
   * difference of an interior-class element is delta = L (q^k - q^{k-1}) and
   *   ||delta||^2_M = J ||R (q^k - q^{k-1})||^2,  R^T R = L^T (W (x) M1 (x) M1) L
   * (W = diag(comp_w), M1 the 1D reference mass): a gram_kc x gram_kc
   * triangle instead of the two sum-factorised mass passes over the volume.
   * q_store keeps every element's neighbour face scalars q (gram_kc per
   * element, tile-major) and is rewritten by every sweep; the kernel uses the
   * stored q^{k-1} only when state->iters > 0, i.e. from the second sweep of
   * a solve on (the first sweep, and tiles with a boundary-class element,
   * take the direct norm).  Contract: between two sweeps of one solve the
   * caller changes neither s nor the operators. */
  double* q_store;            /* [n_tiles_local][tile elems * gram_kc] or NULL (kernel-internal order within a tile) */
  const double* gram_R;       /* [gram_kc][gram_kc] row-major upper-triangular R of the interior class, kernel column order (coupled faces ascending, face nodes) */
  int32_t gram_kc;            /* ihdg_sweep_gram_kc(args), 0 = off */
  int32_t pad2;
  /* Parallel finalize (k_sweep_ws with finalize = 1; both NULL = the
   * single-CTA finalize): the kernel is launched cooperatively, every CTA
   * reduces a share of the element-layer rows of the tile partials into
   * layer_sums after a grid barrier on grid_bar, and the last CTA sums the
   * layer sums -- the order of ihdg_finalize, so the norms are identical. */
  double* layer_sums;         /* [n_layers_local] */
  uint32_t* grid_bar;         /* [2] (arrival count, generation), zero before first use; left reusable */
  /* Per-element operators ("GEMV mode", variable coefficients, SURVEY.md 8f
   * row 1; generic kernel): the operator class of a local element is its
   * index, and with raw_blocks > 0 the neighbour data are raw face-node
   * values instead of weighted scalars: column (f, j, n) of LT holds
   * u_src[raw_comp[f][j]][node n of the shared face] with src = the
   * neighbour across f (j < 2) or the element itself (j >= 2, iHDG-I), so
   * LT is [Nel_local][2d * raw_blocks * (p+1)^(d-1)][NV]. */
  int32_t per_element;
  int32_t raw_blocks;         /* 0 (weighted scalars), 2 or 4 */
  int32_t raw_comp[IHDG_MAX_FACE][4];
} ihdg_sweep_args;

/* K5: ||u - u^e||_{L2(Omega)}^2 per tile by (p+2)^d Gauss quadrature
 * (l2_error), fixed-order tile partials.  mode 0: the
 * initial iterate (state->last_err := error, status untouched).  mode 1:
 * after a sweep with finalize = 0; the last CTA reduces the sweep's
 * successive partials and the error partials and applies the exact-solution
 * stopping rule |e_k - e_{k-1}| < tol; divergence and
 * NaN stay on the successive norm.  mode 2: as mode 1 with the
 * vs-direct rule e_k < tol (section 6.3), ue_q = a direct HDG
 * solution at the Gauss points. */
typedef struct {
  ihdg_geom g;
  const double* u;            /* ghost-padded state */
  const double* ue_q;         /* [Nel_local][ncomp][nq^dim] exact solution at the Gauss points */
  const double* vq;           /* [nq][N1] nodal basis at the Gauss points */
  const double* wq;           /* [nq] Gauss weights on [-1,1] */
  double* err_partials;       /* [ihdg_error_tile_count(g)] */
  const double* succ_partials;/* the sweep's tile partials (mode 1) */
  int64_t n_succ;             /* their count */
  ihdg_iter_state* state;
  double* norm_hist;          /* successive norms [max_iters] or NULL */
  double* err_hist;           /* errors [max_iters] or NULL */
  double comp_w[IHDG_MAX_COMP];
  double jac;
  int32_t nq;
  int32_t mode;
} ihdg_error_args;

/* K6: diagnostics of iteration.run in diagnostic mode (SPEC.md:320-323,
 * 341-349, 398); not on the sweep path.
 * ihdg_elem_error: per local element e,
 *   err2[e] = J sum_c comp_w[c] ||u_{e,c} - r_{e,c}||^2_{M}  (consistent mass,
 *             M1 = C C^T), flags[e] = (err2[e] < tol^2),
 *   *total  = fixed-order sum of err2 (256 virtual lanes).
 * The element convergence map of SPEC.md:321 / layer_convergence_map
 * is flags with r = the converged HDG solution. */
typedef struct {
  ihdg_geom g;
  const double* u;            /* ghost-padded state */
  const double* r;            /* ghost-padded reference state, same layout */
  const double* chol1d;       /* [N1][N1] lower factor C, row-major */
  double* err2;               /* [Nel_local] */
  uint8_t* flags;             /* [Nel_local] or NULL */
  double* total;              /* [1] or NULL */
  double comp_w[IHDG_MAX_COMP];
  double jac;
  double tol;
} ihdg_elem_error_args;

/* Skeleton energy of a face array t[n_faces][(p+1)^(d-1)] (mesh.py face order,
 * e.g. written by ihdg_extract_trace): e2[f] = Jf_axis(f) ||t_f - t_ref_f||^2_{M_f},
 * M_f = M1 x .. x M1 over the tangential axes; *total = fixed-order sum.
 * Trace energy and the skeleton jump norm are this applied to
 * the trace of u^k - r and to the interior-face jump of u^k. */
typedef struct {
  ihdg_geom g;                /* single rank: layer range = whole axis */
  const double* t;
  const double* t_ref;        /* same shape as t, or NULL (= 0) */
  const double* chol1d;
  double* e2;                 /* [n_faces] */
  double* total;              /* [1] or NULL */
  double jac_face[IHDG_MAX_DIM];
} ihdg_face_energy_args;

/* K3 (multi-rank): reduce the gathered partials, update *state.  The
 * partials are n_tiles values in rows of row_len (one row per element layer
 * of the slowest axis, tile order): each row is summed sequentially, the row
 * sums in a fixed order (256 virtual lanes + a fixed tree) -- the order the
 * fused single-rank finalize uses, so a strip partition (which splits only
 * between layers) gives bit-identical norms.  Multi-rank callers pass the
 * all-reduced layer sums of ihdg_layer_sums with row_len 1. */
typedef struct {
  const double* tile_partials; /* [n_tiles] */
  int64_t n_tiles;
  ihdg_iter_state* state;
  double* norm_hist;
  int64_t row_len;             /* tiles per row (<= 0: 1) */
} ihdg_finalize_args;

/* Halo pack / unpack of a strip partition: only the face-node
 * entries a neighbouring rank's sweep reads cross the wire, not whole layers.
 * For every element of one layer of the ghost-padded state, the element-local
 * DOF entries idx[0..n_idx) (component * (p+1)^d + node of the face the
 * neighbour reads, components with a nonzero face weight) are copied to /
 * from packed[element][n_idx]. */
typedef struct {
  ihdg_geom g;
  double* buf;                /* ghost-padded state */
  double* packed;             /* [layer elems][n_idx] */
  const int32_t* idx;         /* [n_idx] element-local entries (device) */
  int32_t n_idx;
  int32_t layer;              /* 0 ghost_lo, 1 first local, 2 last local, 3 ghost_hi */
} ihdg_halo_args;

/* Single-valued trace on every face, mesh.py face order (mesh.py:89-125).
 * Per axis a: interior face (owner = lower element, normal +e_a)
 *   t = sum_c w_int_own[a][c] u_owner_c|face + sum_c w_int_nbr[a][c] u_nbr_c|face
 * boundary face on the low plane (owner normal -e_a): sum_c w_lo[a][c] u_owner_c
 * boundary face on the high plane (owner normal +e_a): sum_c w_hi[a][c] u_owner_c */
typedef struct {
  ihdg_geom g;                /* single rank: layer range = whole axis */
  const double* u;            /* ghost-padded state */
  double* trace;              /* [n_faces][(p+1)^(d-1)] */
  double w_int_own[IHDG_MAX_DIM][IHDG_MAX_COMP];
  double w_int_nbr[IHDG_MAX_DIM][IHDG_MAX_COMP];
  double w_lo[IHDG_MAX_DIM][IHDG_MAX_COMP];
  double w_hi[IHDG_MAX_DIM][IHDG_MAX_COMP];
} ihdg_trace_args;

int ihdg_abi_version(void);
/* sizeof the ABI structs, for binding self-checks: 0 geom, 1 iter_state,
 * 2 assembly_args, 3 class_apply_args, 4 field_args, 5 quad_args,
 * 6 sweep_args, 7 finalize_args, 8 trace_args, 9 error_args, 10 elem_error_args,
 * 11 face_energy_args, 12 halo_args; -1 otherwise */
int64_t ihdg_struct_size(int32_t which);
const char* ihdg_last_error(void);
/* 1 if the sweep/apply kernels are instantiated for (dim, order, ncomp) */
int ihdg_supported(int32_t dim, int32_t order, int32_t ncomp);
/* elements per sweep tile and the number of tiles of a strip */
int32_t ihdg_tile_elems(int32_t dim, int32_t order, int32_t ncomp);
int64_t ihdg_tile_count(const ihdg_geom* g);

int ihdg_assemble(const ihdg_assembly_args* a, void* stream);
int ihdg_class_apply(const ihdg_class_apply_args* a, void* stream);
int ihdg_eval_field(const ihdg_field_args* a, void* stream);
int ihdg_quad_project(const ihdg_quad_args* a, void* stream);
int ihdg_sweep(const ihdg_sweep_args* a, void* stream);
/* 1 if ihdg_sweep would use one of the streaming kernels (ws / v3 / v4) for
 * these args, 0 if it falls back to the generic kernel */
int ihdg_stream_variant(const ihdg_sweep_args* a);
/* Name of the kernel ihdg_sweep launches for these args under the current
 * selector: "k_sweep_ws" (2D warp-specialised, config 5), "k_sweep_v4"
 * (register-tiled, 3D p=3 scalar: config 4), "k_sweep_v5" (register-tiled, 2D
 * p=4: config 2), "k_sweep_v3" (warp-owned tiles behind a staged ring, config
 * 3), "k_sweep_gemv" (per-element operators), "k_sweep" (generic), or NULL if no kernel is instantiated (static string). */
const char* ihdg_sweep_kernel(const ihdg_sweep_args* a);
/* Process-wide sweep-kernel selector: "auto" (default; the initial value is
 * read from the environment variable IHDG_SWEEP_IMPL), "v3" (skip v4 / v5),
 * "v5" (v5 wherever it applies, without the round model), "ws" / "stream"
 * (skip v3, v4 and v5), "generic" (generic kernel only).
 * IHDG_ERR_ARG for other names. */
int ihdg_set_sweep_impl(const char* name);
/* Columns of the Gram factor R the dispatched kernel takes for these args
 * (q scalars per element, see ihdg_sweep_args.q_store), or 0 if the kernel
 * has no Gram-form norm. */
int ihdg_sweep_gram_kc(const ihdg_sweep_args* a);
/* CUDA-graph replay of sweep batches in ihdg_iterate (default on unless the
 * environment sets IHDG_NO_GRAPH): 1 on, 0 off. */
int ihdg_set_graphs(int on);
int ihdg_finalize(const ihdg_finalize_args* a, void* stream);
/* out[r] = sequential sum of row r of the tile partials [n_rows][row_len]
 * (a rank's layer sums, the inner sums of ihdg_finalize) */
int ihdg_layer_sums(const double* tile_partials, int64_t n_rows, int64_t row_len, double* out, void* stream);
/* halo pack (layer 1/2 -> packed) and unpack (packed -> layer 0/3) */
int ihdg_halo_pack(const ihdg_halo_args* a, void* stream);
int ihdg_halo_unpack(const ihdg_halo_args* a, void* stream);
int ihdg_extract_trace(const ihdg_trace_args* a, void* stream);
/* copy the ghost-padded layer range between two buffers (initial guess) */
int ihdg_copy_state(const ihdg_geom* g, const double* src, double* dst, void* stream);

/* Whole Algorithm-1 loop on one device (single rank, finalize forced on):
 * sweeps alternate buf0 -> buf1 -> buf0 ...; the host polls *state every
 * `batch` sweeps.  On return *state_out holds the final control block and the
 * latest iterate is in buf[state_out->iters % 2].  n_launched (host, may be
 * NULL) receives the number of sweep kernels launched. */
int ihdg_iterate(const ihdg_sweep_args* a, double* buf0, double* buf1, int32_t batch,
                 void* stream, ihdg_iter_state* state_out, int64_t* n_launched);

/* K5 (see ihdg_error_args) and its tile count */
int ihdg_error_norm(const ihdg_error_args* e, void* stream);
int64_t ihdg_error_tile_count(const ihdg_geom* g);
/* ihdg_iterate with the exact-solution stopping rule: every sweep runs with
 * finalize = 0 and is followed by K5 (mode 1) on its output; e->u is set per
 * sweep, e->mode forced to 1 (2 kept).  The caller runs K5 in mode 0 on the initial
 * iterate first (state->last_err).  e->mode 2 selects the vs-direct rule. */
int ihdg_iterate_exact(const ihdg_sweep_args* a, const ihdg_error_args* e, double* buf0, double* buf1,
                       int32_t batch, void* stream, ihdg_iter_state* state_out, int64_t* n_launched);
/* K6 diagnostics (see ihdg_elem_error_args / ihdg_face_energy_args) */
int ihdg_elem_error(const ihdg_elem_error_args* a, void* stream);
int ihdg_face_energy(const ihdg_face_energy_args* a, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* IHDG_H */
