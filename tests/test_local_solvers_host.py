"""Host-side pieces of the local_solvers API (no GPU): neighbour lookup
against mesh.py's connectivity, TraceSnapshot extraction, time configs."""

import numpy as np
import pytest

from paper_1711_01175_b200 import local_solvers as LS
from paper_1711_01175_b200.assembly import face_node_indices
from paper_1711_01175_b200.mesh import build_mesh


@pytest.mark.parametrize("dim,cells,periodic", [(2, [4, 3], False), (3, [3, 2, 4], False), (2, [4, 4], True)])
def test_neighbor_matches_mesh_connectivity(dim, cells, periodic):
    mesh = build_mesh(dim, cells, periodic=periodic)
    nb = mesh.neighbor_elements
    for K in range(mesh.n_elements):
        for f in range(2 * dim):
            assert LS._neighbor(mesh, K, f) == nb[K, f]


def test_trace_snapshot_from_state():
    mesh = build_mesh(2, [3, 3])
    p, m = 2, 3
    n1 = p + 1
    data = np.random.default_rng(0).normal(size=(9, m, n1 * n1))
    snap = LS.TraceSnapshot.from_state(mesh, data, 4, boundary_data=lambda x: x[:, 0])
    assert sorted(snap.neighbor) == [0, 1, 2, 3] and snap.boundary == {}
    # face 1 (+x) of element 4 sees element 5's -x face nodes
    assert np.array_equal(snap.neighbor[1], data[5][:, face_node_indices(2, n1, 0)])
    corner = LS.TraceSnapshot.from_state(mesh, data, 0, boundary_data=lambda x: x[:, 0] + 10 * x[:, 1])
    assert sorted(corner.neighbor) == [1, 3] and sorted(corner.boundary) == [0, 2]
    assert np.allclose(corner.boundary[0], 10 * np.array([0.0, 1 / 6, 1 / 3]))   # x = 0 face, y nodes


def test_time_config():
    assert LS._time_cfg(None).scheme() == (None, "BE")
    assert LS._time_cfg(0.1).scheme() == (0.1, "BE")
    assert LS._time_cfg(("crank-nicolson", 0.2)).scheme() == (0.2, "CN")
    assert LS._time_cfg(("locally-implicit", 0.5)).scheme() == (0.5, "BE")
    with pytest.raises(ValueError):
        LS._time_cfg(("backward-euler", None)).scheme()
