// iHDG-II sweep, version 4: register-tiled sweep for 3D p=3 scalar problems
// (BASELINE config 4: transport on 64^3 hexes, 64 DOFs per element), latency
// hidden by occupancy instead of a shared-memory stage ring.
//
// One warp owns one 8-element tile end to end and there are no helper warps.
// Every lane loads its own DMMA operands straight from global memory, all
// issued before the first use (~30 independent 8/16-byte loads per lane):
//   * s    -> the accumulators (D fragment), u^k -> registers in the same
//             layout (for delta = u^{k+1} - u^k), as 16-byte loads: the DMMA
//             row of (row tile rt, fragment row r) is node 16 (rt>>1) + 2 r +
//             (rt&1), so a lane's two row tiles of one z level are adjacent
//             in memory and a quarter warp reads 128 contiguous bytes;
//   * q    -> the B fragment: lane (element n = lane>>2, kk = lane&3) reads the
//             neighbour face nodes it needs (TraceSnapshot of iterate k); on
//             faces of the axes >= 1 the k index is permuted (face node 4 kk + s
//             in step s) so these are two 16-byte loads per face.
// L (interior class) sits in shared memory in A-fragment order with the same
// row / k permutations, one 16-byte load per pair of row tiles.  u^{k+1} is
// stored from registers (16-byte stores).  The stopping norm
// J |(C^T x C^T x C^T) delta|^2 takes its z pass in registers (a lane holds all
// four z levels of its nodes), writes the result once to a warp-private scratch
// tile, and lane (element, z level) finishes the y and x passes on its 4x4
// block in registers: one shared-memory round trip instead of three.
//
// PF = 4 consecutive warps (a group) own the 4 physical tiles of one logical
// tile (the generic kernel's 32-element tile: one tile partial), combined in
// warp order through a named barrier, so the partial layout and the finalize
// order equal the other kernels'.
//
// HBM per element-DOF: s, u^k (LDG), u^{k+1} (STG) = 24 B; the neighbour face
// nodes are L1/L2 hits (their elements are tiles of this or a nearby warp).
#pragma once

#include <climits>

#include "ihdg_stream.cuh"

namespace ihdg {

// ci-th set bit of the coupled-face mask
__host__ __device__ constexpr int v4_face(int fmask, int ci) {
  int n = 0;
  for (int f = 0; f < 6; ++f)
    if ((fmask >> f) & 1) {
      if (n == ci) return f;
      ++n;
    }
  return -1;
}
__host__ __device__ constexpr int v4_popc(int m) { return m == 0 ? 0 : (m & 1) + v4_popc(m >> 1); }

// FMASK: bit f set = local face f is coupled (compile-time, so the gathers
// and the neighbour selection are straight-line code)
template <int FMASK, int NW, int MINB_ = 1>
struct V4Cfg {
  static constexpr int NCF = v4_popc(FMASK);
  static constexpr int D = 3, N1 = 4, M = 1, NWC = 1, PF = 4;
  static constexpr int E = 8;                     // elements per physical tile (DMMA n)
  static constexpr int NP = 64, NV = 64, NF = 16, NFACE = 6;
  static constexpr int KC = NCF * NF;
  static constexpr int NRT = 8;                   // DMMA row tiles
  static constexpr int KS = KC / 4;               // DMMA k steps (4 per coupled face)
  static constexpr int NT = 32 * NW;
  static constexpr int NG = NW / PF;              // groups (logical tiles in flight) per CTA
  static constexpr int MINB = MINB_;
  static constexpr int ES = 66;                   // scratch element stride: conflict-free 16-byte accesses
  static constexpr int SCR = E * ES;              // warp-private scratch tile (doubles)
  // warp-private u^k staging tile, written only by the TMA unit: element pairs
  // (one 1 KB bulk copy each) at a stride of 132 doubles, so the 16-byte
  // read-back of a quarter warp is conflict-free
  static constexpr int PS = 2 * NV + 4;
  static constexpr int UKS = (E / 2) * PS;
  static constexpr int LFR = NRT * KS * 32;       // L fragments (doubles)
  static constexpr int N_DBL = LFR + NW * (SCR + UKS);
  static constexpr size_t BYTES = (size_t)N_DBL * sizeof(double);
  static_assert(NW % PF == 0 && NG >= 1 && NG <= 15, "one named barrier per group");
  static_assert(MINB * (BYTES + 4096 + 1024) <= 233472, "shared memory over the sm_100a limit");
};

// node of DMMA row (row tile rt, fragment row r)
__host__ __device__ constexpr int v4_row(int rt, int r) { return 16 * (rt >> 1) + 2 * r + (rt & 1); }
// face node of k step s (0..3 within the face block), lane kk, on a face of axis ax
__host__ __device__ constexpr int v4_fnode(int ax, int s, int kk) { return ax == 0 ? 4 * s + kk : 4 * kk + s; }

__device__ __forceinline__ double2 ldcs2(const double* p) { return __ldcs(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }

template <int FMASK, int NW, int MINB_>
__global__ void __launch_bounds__(V4Cfg<FMASK, NW, MINB_>::NT, MINB_) k_sweep_v4(const ihdg_sweep_args a) {
  using C = V4Cfg<FMASK, NW, MINB_>;
  constexpr int NCF = C::NCF;
  constexpr int D = 3, N1 = 4, E = C::E, NV = C::NV, NF = C::NF, NFACE = C::NFACE, PF = C::PF;
  constexpr int KS = C::KS, ES = C::ES;

  extern __shared__ __align__(16) double sm[];
  const double2* lfr_s = reinterpret_cast<const double2*>(sm);

  __shared__ double chol_s[N1 * N1];
  __shared__ int com_s[64];                 // class_of_mask
  __shared__ double part_s[C::NG][2][PF];
  __shared__ int last_s;
  __shared__ __align__(8) uint64_t ubar[NW];   // per warp: u^k tile landed

  ihdg_iter_state* st = a.state;
  pdl_launch_dependents();   // the next launch may start its own prologue

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (lane == 0) {
    mbar_init(&ubar[warp], 1);
    fence_mbar_init();   // visible to the async proxy after the setup barrier below
  }
  Geo geo;
  geo.init(a.g, E * PF);  // logical tile = PF physical tiles = the generic kernel's tile
  const int64_t ls = geo.ls;
  const double* __restrict__ uo = a.u_old + ls * NV;
  double* __restrict__ un = a.u_new + ls * NV;
  const int fast_class = a.class_of_mask[0];

  for (int i = tid; i < N1 * N1; i += blockDim.x) chol_s[i] = a.chol1d[i];
  if (tid < 64) com_s[tid] = a.class_of_mask[tid];
  __syncthreads();
  // interior-class L in DMMA A-fragment order with the row / k permutations:
  // entry ((k * KS + ks) * 32 + l) * 2 + h = L[v4_row(2 k + h, l>>2)][column of (ks, l&3)]
  for (int idx = tid; idx < C::LFR; idx += blockDim.x) {
    const int h = idx & 1, l = (idx >> 1) & 31, fr = idx >> 6;
    const int k = fr / KS, ks = fr - k * KS;
    const int ci = ks >> 2;
    const int f = ci == 0 ? v4_face(FMASK, 0) : (ci == 1 ? v4_face(FMASK, NCF > 1 ? 1 : 0) : v4_face(FMASK, NCF > 2 ? 2 : 0));
    const int row = v4_row(2 * k + h, l >> 2);
    const int col = f * NF + v4_fnode(f >> 1, ks & 3, l & 3);
    sm[idx] = a.LT[((size_t)fast_class * (NFACE * NF) + col) * NV + row];
  }
  __syncthreads();

  // everything above reads only launch-invariant data (operators, tables);
  // the iterate, s and the iteration state belong to the previous launches
  pdl_wait();
  if (st->status != IHDG_RUNNING) return;

  const int grp = warp / PF, sub = warp - grp * PF;
  const int nlog = (int)geo.ntiles;
  const int nlay = (int)(a.g.layer_end - a.g.layer_begin);
  const int lsi = (int)ls;
  const int c0 = (int)a.g.cells[0];
  const int per0 = a.g.periodic[0];
  const int kk = lane & 3;
  const int te = 2 * kk;              // D-fragment columns (elements) of this lane
  const int rsub = lane >> 2;         // D-fragment row inside a row tile; B-fragment element
  double* scr = sm + C::LFR + warp * (C::SCR + C::UKS);
  double* uks = scr + C::SCR;
  FastDiv dsegs0, dc1;
  dsegs0.init((uint32_t)(c0 / E));
  dc1.init((uint32_t)a.g.cells[1]);
  const int segs0 = c0 / E;
  const double cw = a.comp_w[0];

  // per coupled face: weight and this lane's first source node offset inside
  // the neighbour (its face f^1; axes >= 1: 4 consecutive nodes, axis 0: stride 16)
  int bo[NCF];
  double bw[NCF];
#pragma unroll
  for (int ci = 0; ci < NCF; ++ci) {
    const int f = v4_face(FMASK, ci);
    bw[ci] = a.face_w[f][0];
    bo[ci] = face_node_vidx(D, N1, f ^ 1, v4_fnode(f >> 1, 0, kk));
  }
  // tile partial of a logical tile: the group's warps in order.  Called one
  // iteration late (after the next tile's loads are issued), so the group
  // barrier waits while those loads are in flight.
  auto group_partial = [&](int lt_done, int it_done) {
    named_bar_sync(1 + grp, 32 * PF);
    if (sub == 0 && lane == 0) {
      double p = 0.0;
#pragma unroll
      for (int w = 0; w < PF; ++w) p += part_s[grp][it_done & 1][w];
      a.tile_partials[lt_done] = a.jac * p;
    }
  };
  int itn = 0, prev_lt = -1;
  for (int lt = (int)blockIdx.x * C::NG + grp; lt < nlog; lt += (int)gridDim.x * C::NG, ++itn) {
    STile<D> ti;
    ti.init(a.g, lt * PF + sub, E, nlay, lsi, segs0, dsegs0, dc1);
    const int e0 = ti.e0;
    // ---- operand loads, all independent ----
    // acc[k][v] / uk[k][v]: nodes 16 k + 2 rsub + {0, 1} (row tiles 2k, 2k+1) of element te + v
    double2 acc[4][2];
    double b[KS];
    {
      const double* sg = a.s + (int64_t)(e0 + te) * NV + 2 * rsub;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[k][0] = ldcs2(sg + 16 * k);
        acc[k][1] = ldcs2(sg + NV + 16 * k);
      }
    }
    // u^k tile -> the staging tile by the TMA unit (one 1 KB bulk copy per
    // element pair), read back in the epilogue.  The region is never written
    // through the generic proxy, so no proxy fence is needed; the warp's
    // read-back of the previous tile is ordered by __syncwarp.
    __syncwarp();
    if (lane == 0) {
      mbar_arrive_expect_tx(&ubar[warp], (uint32_t)(E * NV * sizeof(double)));
#pragma unroll
      for (int pr = 0; pr < E / 2; ++pr)
        bulk_g2s(uks + pr * C::PS, uo + (int64_t)(e0 + 2 * pr) * NV, (uint32_t)(2 * NV * sizeof(double)), &ubar[warp]);
    }
    {
      // neighbour of element rsub across each face (a missing one reads the
      // element itself with weight 0: branch-free gathers)
      constexpr int NONE = INT_MIN;   // ghost-layer neighbours have negative local indices
      const int i = ti.i0 + rsub;
#pragma unroll
      for (int ci = 0; ci < NCF; ++ci) {
        const int f = v4_face(FMASK, ci);   // compile-time after unrolling
        int nb;
        if (f == 0) nb = (!per0 && i == 0) ? NONE : e0 + rsub + (i > 0 ? -1 : c0 - 1);
        else if (f == 1) nb = (!per0 && i == c0 - 1) ? NONE : e0 + rsub + (i < c0 - 1 ? 1 : -(c0 - 1));
        else nb = ti.has[f] ? e0 + rsub + ti.off[f] : NONE;
        const double w = nb != NONE ? bw[ci] : 0.0;
        const double* src = uo + (int64_t)(nb != NONE ? nb : e0 + rsub) * NV + bo[ci];
        if (f < 2) {   // x face: nodes (j = kk, k = s), stride 16
#pragma unroll
          for (int s = 0; s < 4; ++s) b[4 * ci + s] = w * __ldg(src + 16 * s);
        } else {       // y / z face: four consecutive nodes
          const double2 g0 = ldg2(src), g1 = ldg2(src + 2);
          b[4 * ci + 0] = w * g0.x;
          b[4 * ci + 1] = w * g0.y;
          b[4 * ci + 2] = w * g1.x;
          b[4 * ci + 3] = w * g1.y;
        }
      }
    }
    if (prev_lt >= 0) group_partial(prev_lt, itn - 1);
    // ---- operator classes of the tile ----
    const int mycls = com_s[ti.mask(rsub, c0, per0)];
    const int fast = __all_sync(0xffffffffu, mycls == fast_class);
    if (fast) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 l2 = lfr_s[(k * KS + ks) * 32 + lane];
          // row tile 2k holds the .x halves, 2k+1 the .y halves, of both elements
          dmma_8x8x4(acc[k][0].x, acc[k][1].x, l2.x, b[ks]);
          dmma_8x8x4(acc[k][0].y, acc[k][1].y, l2.y, b[ks]);
        }
      }
    } else {
      // one masked pass per operator class present in the tile
      unsigned cset = (mycls >= 0 && mycls < 32) ? (1u << mycls) : 0u;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cset |= __shfl_xor_sync(0xffffffffu, cset, o);
      for (unsigned rem = cset; rem != 0u; rem &= rem - 1u) {
        const int c = __ffs(rem) - 1;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const double bb = (mycls == c) ? b[ks] : 0.0;
          const int f = v4_face(FMASK, ks >> 2);
          const int col = f * NF + v4_fnode(f >> 1, ks & 3, kk);
          const double* Lc = a.LT + ((size_t)c * (NFACE * NF) + col) * NV;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            dmma_8x8x4(acc[k][0].x, acc[k][1].x, __ldg(Lc + v4_row(2 * k, rsub)), bb);
            dmma_8x8x4(acc[k][0].y, acc[k][1].y, __ldg(Lc + v4_row(2 * k + 1, rsub)), bb);
          }
        }
      }
    }
    // ---- u^{k+1} -> global (16-byte stores), delta in registers ----
    {
      double* ug = un + (int64_t)(e0 + te) * NV + 2 * rsub;
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int v = 0; v < 2; ++v)
          __stcs(reinterpret_cast<double2*>(ug + v * NV + 16 * k), acc[k][v]);
    }
    mbar_wait(&ubar[warp], itn & 1);   // the u^k tile has landed
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const double2 u2 = *reinterpret_cast<const double2*>(uks + kk * C::PS + v * NV + 16 * k + 2 * rsub);
        acc[k][v].x -= u2.x;
        acc[k][v].y -= u2.y;
      }
    // ||delta||_M^2 = J |(C^T x C^T x C^T) delta|^2, M1 = C C^T.  z pass in
    // registers: y_k = sum_{k' >= k} C[k'][k] x_k' along the four z levels
    // (the block reads of the previous tile finished before this tile's __syncwarp above)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double yx = 0.0, yy = 0.0;
#pragma unroll
        for (int kp = k; kp < 4; ++kp) {
          yx = fma(chol_s[kp * N1 + k], acc[kp][v].x, yx);
          yy = fma(chol_s[kp * N1 + k], acc[kp][v].y, yy);
        }
        *reinterpret_cast<double2*>(scr + (te + v) * ES + 16 * k + 2 * rsub) = make_double2(yx, yy);
      }
    }
    __syncwarp();
    // lane (element t = lane & 7, z level k = lane >> 3): y then x pass on its 4x4 block
    double nsum = 0.0;
    {
      const double* blk = scr + (lane & 7) * ES + 16 * (lane >> 3);
      double x[4][4];   // [j][i]
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 p0 = *reinterpret_cast<const double2*>(blk + 4 * j);
        const double2 p1 = *reinterpret_cast<const double2*>(blk + 4 * j + 2);
        x[j][0] = p0.x;
        x[j][1] = p0.y;
        x[j][2] = p1.x;
        x[j][3] = p1.y;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double y = 0.0;
#pragma unroll
          for (int jp = j; jp < 4; ++jp) y = fma(chol_s[jp * N1 + j], x[jp][i], y);
          x[j][i] = y;   // in place: row j is final once rows >= j were read
        }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double sq = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double y = 0.0;
#pragma unroll
          for (int ip = i; ip < 4; ++ip) y = fma(chol_s[ip * N1 + i], x[j][ip], y);
          sq = fma(y, y, sq);
        }
        nsum += sq;
      }
      nsum *= cw;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, o);
    if (lane == 0) part_s[grp][itn & 1][sub] = nsum;
    prev_lt = lt;
  }
  if (prev_lt >= 0) group_partial(prev_lt, itn - 1);

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
