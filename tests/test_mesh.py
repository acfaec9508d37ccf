"""Mesh numbering contract, pinned against the reference's own mesh.py
(fixtures from tests/golden/make_golden.py) and SPEC.md:45-68 examples."""

import os

import numpy as np
import pytest

from oracle.ihdg_oracle import structured_neighbors
from paper_1711_01175_b200.mesh import BOUNDARY, build_mesh, classify_boundary_faces

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "mesh_reference.npz"))
CASES = range(int(GOLD["ncases"]))
BETAS = {1: [1.0], 2: [1.0, -0.5], 3: [0.2, 0.2, 0.2]}


@pytest.mark.parametrize("ci", CASES)
def test_connectivity_matches_reference(ci):
    k = f"c{ci}"
    dim, cells = int(GOLD[f"{k}_dim"]), list(GOLD[f"{k}_cells"])
    m = build_mesh(dim, cells)
    assert np.array_equal(m.element_to_faces, GOLD[f"{k}_element_to_faces"])
    assert np.array_equal(m.neighbor_elements, GOLD[f"{k}_neighbor_elements"])
    assert np.array_equal(m.neighbor_faces, GOLD[f"{k}_neighbor_faces"])
    assert np.array_equal(m.face_axis, GOLD[f"{k}_face_axis"])
    assert np.array_equal(m.face_owner, GOLD[f"{k}_face_owner"])
    assert np.array_equal(m.face_neighbor, GOLD[f"{k}_face_neighbor"])
    # the oracle's index-arithmetic neighbours agree with the reference too
    assert np.array_equal(structured_neighbors(cells), GOLD[f"{k}_neighbor_elements"])


@pytest.mark.parametrize("ci", CASES)
def test_geometry_matches_reference_bitwise(ci):
    k = f"c{ci}"
    dim, cells = int(GOLD[f"{k}_dim"]), list(GOLD[f"{k}_cells"])
    m = build_mesh(dim, cells)
    ref1d = GOLD["ref1d"]
    normals = np.array([f.normal for f in m.faces])
    cents = np.array([f.centroid for f in m.faces])
    meas = np.array([f.measure for f in m.faces])
    assert np.array_equal(normals, GOLD[f"{k}_face_normal"])
    assert np.array_equal(cents, GOLD[f"{k}_face_centroid"])
    assert np.array_equal(meas, GOLD[f"{k}_face_measure"])
    fp = np.array([m.face_points(f, ref1d[1:3]) for f in range(m.n_faces)])
    assert np.array_equal(fp, GOLD[f"{k}_face_points"])
    ep = m.all_element_points([ref1d] * dim)
    assert np.array_equal(ep, GOLD[f"{k}_element_points"])
    assert m.boundary_surface_measure() == float(GOLD[f"{k}_boundary_measure"])
    b = np.array(BETAS[dim])
    tagged = classify_boundary_faces(m, lambda x: np.tile(b, (x.shape[0], 1)))
    assert [f.tag for f in tagged.faces] == list(GOLD[f"{k}_tags"])


def test_spec_examples():
    m = build_mesh(2, [4, 4])
    assert m.n_elements == 16 and m.n_faces == 40
    assert len(m.interior_faces) == 24 and len(m.boundary_faces) == 16
    m = build_mesh(3, [2, 2, 2])
    assert m.n_elements == 8 and m.n_faces == 36
    m = build_mesh(1, [5], (np.zeros(1), np.ones(1)))
    assert m.n_elements == 5 and m.n_faces == 6 and np.isclose(m.h[0], 0.2)
    for n in (3, 7):
        assert build_mesh(2, [n, n]).n_faces == 2 * n * (n + 1)
        assert build_mesh(3, [n, n, n]).n_faces == 3 * n * n * (n + 1)


def test_errors():
    with pytest.raises(ValueError):
        build_mesh(4, [2])
    with pytest.raises(ValueError):
        build_mesh(2, [0, 3])
    with pytest.raises(ValueError):
        build_mesh(2, [2, 2], (np.zeros(2), np.array([1.0, 0.0])))


def test_invariants():
    m = build_mesh(3, [3, 4, 2])
    assert abs(m.boundary_surface_measure() - 6.0) < 1e-12
    for f in m.faces:
        assert abs(np.linalg.norm(f.normal) - 1.0) < 1e-14
    ref = np.array([-0.7, 0.1, 0.9])
    for fid in m.interior_faces:
        f = m.faces[fid]
        lo = m.element_face_points(f.owner, 2 * f.axis + 1, ref)
        hi = m.element_face_points(f.neighbor, 2 * f.axis + 0, ref)
        assert np.max(np.abs(lo - hi)) <= 1e-14
    m2 = build_mesh(3, [3, 4, 2])
    assert np.array_equal(m.neighbor_elements, m2.neighbor_elements)


def test_periodic_option():
    m = build_mesh(2, [4, 3], periodic=True)
    assert m.n_faces == 2 * 12
    assert len(m.boundary_faces) == 0
    nb = m.neighbor_elements
    assert (nb != BOUNDARY).all()
    assert np.array_equal(nb, structured_neighbors([4, 3], [True, True]))
    # every element's high neighbour sees it as its low neighbour
    for e in range(m.n_elements):
        for a in range(2):
            assert nb[nb[e, 2 * a + 1], 2 * a] == e
    assert m.boundary_surface_measure() == 0.0


def test_large_mesh_is_lazy():
    m = build_mesh(2, [2048, 2048])
    assert m.n_faces == 2 * 2048 * 2049
    f = m.faces[m.n_faces - 1]
    assert f.neighbor == BOUNDARY and f.axis == 1
