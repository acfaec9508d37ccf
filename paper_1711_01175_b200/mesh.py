"""Uniform structured tensor-product meshes.

Same API and numbering contract as the reference ``ihdg.mesh``
(pkg/src/ihdg/mesh.py), rebuilt for meshes with millions of elements:

- elements lexicographic, axis 0 fastest (mesh.py:73-75, 144-149);
- local face slot ``2*axis + side``, side 0 = low face with normal -e_axis
  (mesh.py:43-48);
- faces numbered axis by axis, plane by plane, tangential multi-index with the
  smallest tangential axis fastest (mesh.py:89-125); a face is owned by its
  lower element when it has one (normal +e_axis), else by the upper element
  (normal -e_axis) (mesh.py:109-116);
- owner and neighbour enumerate face points in the same order (mesh.py:166-187).

Differences (additive, defaults unchanged): connectivity arrays are built
vectorised and lazily, ``faces`` is a lazy sequence of ``Face`` records, and
``periodic=`` (per axis) wraps the mesh; on a periodic axis the plane-0 face is
the wrap face, owned by the last element with the first one as neighbour
(SURVEY.md Appendix B.6).  The GPU sweep never needs the arrays: it derives
neighbours from the structured strides.
"""

from __future__ import annotations

import copy
from dataclasses import dataclass
from functools import cached_property

import numpy as np

BOUNDARY = -1

BOUNDARY_TAGS = ("inflow", "outflow", "wall", "dirichlet")

__all__ = ["BOUNDARY", "BOUNDARY_TAGS", "Face", "StructuredMesh", "build_mesh",
           "classify_boundary_faces"]


@dataclass
class Face:
    """One mesh face: owner side carries the outward unit normal (mesh.py:19-30)."""

    index: int
    axis: int
    owner: int
    neighbor: int  # element id or BOUNDARY
    normal: np.ndarray
    centroid: np.ndarray
    measure: float
    tag: str = ""


class _FaceList:
    """Lazy, indexable view of all faces (records built on access)."""

    def __init__(self, mesh: "StructuredMesh"):
        self._mesh = mesh
        self._tags: dict[int, str] = {}

    def __len__(self) -> int:
        return self._mesh.n_faces

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]

    def __getitem__(self, fid):
        if isinstance(fid, slice):
            return [self[i] for i in range(*fid.indices(len(self)))]
        fid = int(fid)
        if fid < 0:
            fid += len(self)
        if not 0 <= fid < len(self):
            raise IndexError(fid)
        return self._mesh._face_record(fid, self._tags.get(fid, ""))

    def _copy(self, mesh):
        new = _FaceList(mesh)
        new._tags = dict(self._tags)
        return new


class StructuredMesh:
    """Tensor-product tessellation of ``[lo, hi]`` with ``cells_per_dim`` cells."""

    def __init__(self, dim, cells_per_dim, box, periodic=False):
        if dim not in (1, 2, 3):
            raise ValueError(f"dim must be 1, 2 or 3, got {dim}")
        cells = tuple(int(n) for n in np.atleast_1d(cells_per_dim))
        if len(cells) == 1 and dim > 1:
            cells = cells * dim
        if len(cells) != dim:
            raise ValueError(f"need {dim} cell counts, got {cells}")
        if any(n < 1 for n in cells):
            raise ValueError(f"cell counts must be positive, got {cells}")
        lo = np.asarray(box[0], dtype=float).reshape(dim)
        hi = np.asarray(box[1], dtype=float).reshape(dim)
        if np.any(hi <= lo):
            raise ValueError(f"degenerate box: lo={lo}, hi={hi}")
        per = np.broadcast_to(np.asarray(periodic, dtype=bool), (dim,)).copy()
        self.dim = dim
        self.cells = cells
        self.lo = lo
        self.hi = hi
        self.h = (hi - lo) / np.array(cells, dtype=float)
        self.n_elements = int(np.prod(cells))
        self.periodic = tuple(bool(x) for x in per)
        self._strides = np.ones(dim, dtype=np.int64)
        for a in range(1, dim):
            self._strides[a] = self._strides[a - 1] * cells[a - 1]
        # faces per axis: planes x tangential count
        self._planes = [cells[a] + (0 if self.periodic[a] else 1) for a in range(dim)]
        self._ntan = [int(np.prod([cells[b] for b in range(dim) if b != a])) for a in range(dim)]
        off = [0]
        for a in range(dim):
            off.append(off[-1] + self._planes[a] * self._ntan[a])
        self._face_offset = off
        self.n_faces = off[-1]
        self.faces = _FaceList(self)

    # -- construction (vectorised) -----------------------------------------

    def _axis_face_elements(self, a):
        """(owner, neighbor, side, plane, tangential multi-index) per face of axis a."""
        dim, cells = self.dim, self.cells
        tang = [b for b in range(dim) if b != a]
        nplanes, nt = self._planes[a], self._ntan[a]
        plane = np.repeat(np.arange(nplanes, dtype=np.int64), nt)
        tl = np.tile(np.arange(nt, dtype=np.int64), nplanes)
        tidx = {}
        rem = tl.copy()
        for b in tang:  # smallest tangential axis fastest
            tidx[b] = rem % cells[b]
            rem //= cells[b]
        base = np.zeros_like(tl)
        for b in tang:
            base += tidx[b] * self._strides[b]
        sa = self._strides[a]
        if self.periodic[a]:
            lower = np.where(plane > 0, plane - 1, cells[a] - 1)
            owner = base + lower * sa
            neighbor = base + plane * sa
            side = np.ones_like(plane)
        else:
            has_lower = plane > 0
            has_upper = plane < cells[a]
            owner = np.where(has_lower, base + (plane - 1) * sa, base + plane * sa)
            neighbor = np.where(has_lower & has_upper, base + plane * sa, BOUNDARY)
            side = np.where(has_lower, 1, 0)
        return owner, neighbor, side, plane, tidx

    @cached_property
    def _face_arrays(self):
        owners, nbrs, sides, axes = [], [], [], []
        for a in range(self.dim):
            o, n, s, _, _ = self._axis_face_elements(a)
            owners.append(o)
            nbrs.append(n)
            sides.append(s)
            axes.append(np.full(o.shape, a, dtype=np.int64))
        return (np.concatenate(owners), np.concatenate(nbrs), np.concatenate(sides),
                np.concatenate(axes))

    @property
    def face_owner(self) -> np.ndarray:
        return self._face_arrays[0]

    @property
    def face_neighbor(self) -> np.ndarray:
        return self._face_arrays[1]

    @property
    def face_axis(self) -> np.ndarray:
        return self._face_arrays[3]

    @cached_property
    def _connectivity(self):
        dim, nel = self.dim, self.n_elements
        e2f = np.full((nel, 2 * dim), -1, dtype=np.int64)
        nbr_e = np.full((nel, 2 * dim), BOUNDARY, dtype=np.int64)
        nbr_f = np.full((nel, 2 * dim), BOUNDARY, dtype=np.int64)
        for a in range(dim):
            o, n, s, _, _ = self._axis_face_elements(a)
            fid = self._face_offset[a] + np.arange(o.size, dtype=np.int64)
            e2f[o, 2 * a + s] = fid
            inter = n != BOUNDARY
            e2f[n[inter], 2 * a + 0] = fid[inter]
            nbr_e[o[inter], 2 * a + 1] = n[inter]
            nbr_f[o[inter], 2 * a + 1] = 2 * a + 0
            nbr_e[n[inter], 2 * a + 0] = o[inter]
            nbr_f[n[inter], 2 * a + 0] = 2 * a + 1
        return e2f, nbr_e, nbr_f

    @property
    def element_to_faces(self) -> np.ndarray:
        return self._connectivity[0]

    @property
    def neighbor_elements(self) -> np.ndarray:
        return self._connectivity[1]

    @property
    def neighbor_faces(self) -> np.ndarray:
        return self._connectivity[2]

    @cached_property
    def interior_faces(self) -> list:
        return np.nonzero(self.face_neighbor != BOUNDARY)[0].tolist()

    @cached_property
    def boundary_faces(self) -> list:
        return np.nonzero(self.face_neighbor == BOUNDARY)[0].tolist()

    def _face_record(self, fid: int, tag: str) -> Face:
        a = int(np.searchsorted(self._face_offset, fid, side="right") - 1)
        lf = fid - self._face_offset[a]
        plane, tl = divmod(lf, self._ntan[a])
        tang = [b for b in range(self.dim) if b != a]
        tidx = {}
        for b in tang:
            tidx[b] = tl % self.cells[b]
            tl //= self.cells[b]
        base = sum(int(tidx[b]) * int(self._strides[b]) for b in tang)
        sa = int(self._strides[a])
        if self.periodic[a]:
            lower = plane - 1 if plane > 0 else self.cells[a] - 1
            owner, neighbor, sign = base + lower * sa, base + plane * sa, 1.0
        elif plane > 0:
            owner = base + (plane - 1) * sa
            neighbor = base + plane * sa if plane < self.cells[a] else BOUNDARY
            sign = 1.0
        else:
            owner, neighbor, sign = base, BOUNDARY, -1.0
        normal = np.zeros(self.dim)
        normal[a] = sign
        centroid = np.empty(self.dim)
        centroid[a] = self.lo[a] + plane * self.h[a]
        for b in tang:
            centroid[b] = self.lo[b] + (tidx[b] + 0.5) * self.h[b]
        measure = float(np.prod([self.h[b] for b in tang])) if tang else 1.0
        return Face(int(fid), a, int(owner), int(neighbor), normal, centroid, measure, tag)

    # -- geometry queries (mesh.py:144-211) --------------------------------

    def element_multi_index(self, e):
        return tuple(int(e // self._strides[a] % self.cells[a]) for a in range(self.dim))

    def element_origin(self, e):
        return self.lo + np.array(self.element_multi_index(e)) * self.h

    def element_points(self, e, ref1d):
        """Tensor grid in element ``e``; ``ref1d[a]`` per-axis reference coords."""
        orig = self.element_origin(e)
        axes = [orig[a] + 0.5 * self.h[a] * (np.asarray(ref1d[a]) + 1.0) for a in range(self.dim)]
        return _tensor_points(axes)

    def all_element_points(self, ref1d) -> np.ndarray:
        """(Nel, npts, dim) tensor points of every element (vectorised)."""
        nel = self.n_elements
        e = np.arange(nel, dtype=np.int64)
        per_axis = []
        for a in range(self.dim):
            ia = (e // self._strides[a]) % self.cells[a]
            orig = self.lo[a] + ia * self.h[a]  # element_origin, mesh.py:151-153
            per_axis.append(orig[:, None] + 0.5 * self.h[a] * (np.asarray(ref1d[a])[None, :] + 1.0))
        npts = int(np.prod([len(r) for r in ref1d]))
        out = np.empty((nel, npts, self.dim))
        for a in range(self.dim):
            shape = [1] * self.dim
            shape[self.dim - 1 - a] = len(ref1d[a])
            grid = np.broadcast_to(
                per_axis[a].reshape((nel,) + tuple(shape)),
                (nel,) + tuple(len(ref1d[b]) for b in reversed(range(self.dim))))
            out[:, :, a] = grid.reshape(nel, npts)
        return out

    def face_points(self, fid, ref1d):
        """Points on face ``fid`` (shared ordering; ``ref1d`` is one 1D array)."""
        face = self.faces[fid]
        tang = [a for a in range(self.dim) if a != face.axis]
        if not tang:
            return face.centroid.reshape(1, self.dim)
        axes = [face.centroid[a] - 0.5 * self.h[a] + 0.5 * self.h[a] * (np.asarray(ref1d) + 1.0)
                for a in tang]
        pts = _tensor_points(axes)
        out = np.empty((pts.shape[0], self.dim))
        out[:, face.axis] = face.centroid[face.axis]
        for k, a in enumerate(tang):
            out[:, a] = pts[:, k]
        return out

    def element_face_points(self, e, local_face, ref1d):
        return self.face_points(self.element_to_faces[e, local_face], ref1d)

    def boundary_surface_measure(self):
        total = 0.0
        for a in range(self.dim):
            if self.periodic[a]:
                continue
            meas = float(np.prod([self.h[b] for b in range(self.dim) if b != a])) if self.dim > 1 else 1.0
            total += 2 * self._ntan[a] * meas
        return total

    def tag_boundary(self, tag):
        """Return a copy with every boundary face tagged ``tag``."""
        if tag not in BOUNDARY_TAGS:
            raise ValueError(f"unknown boundary tag {tag!r}")
        tagged = copy.copy(self)
        tagged.faces = self.faces._copy(tagged)
        for fid in self.boundary_faces:
            tagged.faces._tags[fid] = tag
        return tagged


def _tensor_points(axes):
    grids = np.meshgrid(*axes, indexing="ij")
    cols = [g.ravel(order="F") for g in grids]  # axis 0 fastest
    return np.stack(cols, axis=-1)


def build_mesh(dim, cells_per_dim, box=None, periodic=False):
    """Build a StructuredMesh; ``box`` defaults to the unit square/cube."""
    if box is None:
        box = (np.zeros(dim), np.ones(dim))
    return StructuredMesh(dim, cells_per_dim, box, periodic=periodic)


def classify_boundary_faces(mesh, beta, n_quad=4):
    """Tag boundary faces by the sign of ``beta . n`` at Gauss points
    (mesh.py:221-251): all negative -> "inflow", none negative -> "outflow"
    (beta.n = 0 counts as outflow), otherwise "mixed" with a per-point mask."""
    from numpy.polynomial.legendre import leggauss

    ref, _ = leggauss(n_quad)
    tagged = copy.copy(mesh)
    tagged.faces = mesh.faces._copy(tagged)
    masks = {}
    for fid in mesh.boundary_faces:
        face = mesh.faces[fid]
        pts = mesh.face_points(fid, ref)
        bn = np.asarray(beta(pts)) @ face.normal
        mask = bn < 0.0
        masks[fid] = mask
        if mask.all():
            tagged.faces._tags[fid] = "inflow"
        elif not mask.any():
            tagged.faces._tags[fid] = "outflow"
        else:
            tagged.faces._tags[fid] = "mixed"
    tagged.inflow_masks = masks
    return tagged
