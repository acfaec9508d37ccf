// Shared device helpers for the iHDG-II sweep kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ihdg.h"

namespace ihdg {

template <int B, int E>
struct Pow {
  static constexpr int v = B * Pow<B, E - 1>::v;
};
template <int B>
struct Pow<B, 0> {
  static constexpr int v = 1;
};

constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }
__host__ __device__ inline int ipow(int b, int e) {
  int r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}
constexpr int cmin(int a, int b) { return a < b ? a : b; }
constexpr int cmax(int a, int b) { return a > b ? a : b; }

// Compile-time sizes of one (dim, p+1, m) instantiation.
template <int D, int N1, int M>
struct Cfg {
  static constexpr int NP = Pow<N1, D>::v;        // nodes per element
  static constexpr int NV = M * NP;               // volume DOFs per element
  static constexpr int NF = Pow<N1, D - 1>::v;    // nodes per face
  static constexpr int NFACE = 2 * D;
  static constexpr int KIN = NFACE * NF;          // neighbour face scalars per element
  static constexpr int RP = cmin(round_up(NV, 32), 256);  // threads along rows
  static constexpr int G = cmax(1, 128 / RP);             // element groups
  static constexpr int NT = RP * G;                       // threads per CTA
  static constexpr int J = NV <= 160 ? 16 : (NV <= 256 ? 8 : 4);  // accumulators / thread
  static constexpr int TE = J * G;                        // elements per tile
};

// Runtime view of the strip geometry.
struct Geo {
  int D;
  int64_t c[3];
  int per[3];
  int64_t stride[3];
  int64_t lb, le, ls, nloc, nlay;
  int64_t tile_len;   // elements per tile row (a layer, or the strip in 1D)
  int64_t segs;       // tiles per tile row
  int64_t ntiles;

  __host__ __device__ void init(const ihdg_geom& g, int TE) {
    D = g.dim;
    for (int a = 0; a < 3; ++a) {
      c[a] = a < D ? g.cells[a] : 1;
      per[a] = a < D ? g.periodic[a] : 0;
    }
    stride[0] = 1;
    for (int a = 1; a < 3; ++a) stride[a] = stride[a - 1] * c[a - 1];
    ls = stride[D - 1];
    lb = g.layer_begin;
    le = g.layer_end;
    nlay = le - lb;
    nloc = nlay * ls;
    tile_len = (D == 1) ? nloc : ls;
    segs = (tile_len + TE - 1) / TE;
    ntiles = (D == 1) ? segs : nlay * segs;
  }

  // tile -> [e0, e0 + n) local element range
  __host__ __device__ void tile_range(int64_t tile, int TE, int64_t& e0, int& n) const {
    int64_t row = tile / segs, seg = tile % segs;
    e0 = row * tile_len + seg * TE;
    int64_t rem = tile_len - seg * TE;
    n = (int)(rem < TE ? rem : TE);
  }

  __device__ void multi_index(int64_t e, int64_t idx[3]) const {
    for (int a = 0; a < D - 1; ++a) idx[a] = (e / stride[a]) % c[a];
    idx[D - 1] = lb + e / ls;
  }

  // Neighbour across local face f = 2*axis + side (mesh.py:44-48 slot
  // convention).  Returns false on a physical boundary.  The neighbour's local
  // index may be -ls..-1 (low ghost layer) or nloc..nloc+ls-1 (high ghost).
  __device__ bool neighbor(int64_t e, const int64_t idx[3], int f, int64_t& nb) const {
    const int a = f >> 1;
    const int s = f & 1;
    int64_t j = idx[a] + (s ? 1 : -1);
    if (j < 0) {
      if (!per[a]) return false;
      j = c[a] - 1;
    } else if (j >= c[a]) {
      if (!per[a]) return false;
      j = 0;
    }
    if (a < D - 1) {
      nb = e + (j - idx[a]) * stride[a];
    } else {
      int64_t l = j - lb;
      int64_t in_layer = e % ls;
      if (l >= 0 && l < nlay) nb = l * ls + in_layer;
      else nb = (s ? nlay : -1) * ls + in_layer;
    }
    return true;
  }
};

// Per-tile neighbour geometry for tiles that lie inside one axis-0 row
// (requires cells[0] % TE == 0).  Everything the sweep needs per element is
// derived from the first element with integer compares; the int64 div/mod
// of Geo::multi_index runs once per tile instead of once per element-face.
struct TileInfo {
  int64_t e0;       // first local element
  int nt;           // elements in the tile
  int i0;           // axis-0 index of the first element
  int c0;           // cells along axis 0
  int per0;         // axis 0 periodic
  int has[6];       // face f (axis >= 1) has a neighbour (uniform over the tile)
  int64_t off[6];   // neighbour element offset for faces of axis >= 1

  __device__ void init(const Geo& g, int64_t tile, int TE) {
    g.tile_range(tile, TE, e0, nt);
    int64_t idx[3];
    g.multi_index(e0, idx);
    i0 = (int)idx[0];
    c0 = (int)g.c[0];
    per0 = g.per[0];
    for (int f = 0; f < 6; ++f) {
      has[f] = 0;
      off[f] = 0;
    }
    for (int f = 2; f < 2 * g.D; ++f) {
      int64_t nb;
      has[f] = g.neighbor(e0, idx, f, nb) ? 1 : 0;
      off[f] = has[f] ? nb - e0 : 0;
    }
  }
  // missing-neighbour mask of tile element t
  __device__ int mask(int t, int D) const {
    int m = 0;
    const int i = i0 + t;
    if (!per0) {
      if (i == 0) m |= 1;
      if (i == c0 - 1) m |= 2;
    }
    for (int f = 2; f < 2 * D; ++f)
      if (!has[f]) m |= 1 << f;
    return m;
  }
  // local index of the neighbour of tile element t across face f (valid only
  // when the mask bit is clear)
  __device__ int64_t nbr(int t, int f) const {
    const int64_t e = e0 + t;
    if (f >= 2) return e + off[f];
    const int i = i0 + t;
    if (f == 0) return i > 0 ? e - 1 : e + (c0 - 1);
    return i < c0 - 1 ? e + 1 : e - (c0 - 1);
  }
};

// Volume index of node n of local face f (tangential axes increasing, the
// smallest fastest: mesh.py:166-187 shared ordering; nodes lexicographic with
// axis 0 fastest: mesh.py:155-164).
__host__ __device__ inline int face_node_vidx(int D, int N1, int f, int n) {
  const int a = f >> 1;
  const int s = f & 1;
  int v = 0, mul = 1;
  for (int b = 0; b < D; ++b) {
    int ib;
    if (b == a) {
      ib = s ? N1 - 1 : 0;
    } else {
      ib = n % N1;
      n /= N1;
    }
    v += ib * mul;
    mul *= N1;
  }
  return v;
}

}  // namespace ihdg
