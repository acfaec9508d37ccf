"""Generate golden fixtures from the reference package itself.

Run in the build container (needs /root/reference, read-only):

    python tests/golden/make_golden.py

The only executable part of the reference is ``ihdg.mesh``
(pkg/src/ihdg/mesh.py); it is the numbering contract of the whole sweep
(SURVEY.md section 8a rows a1-a3).  This script imports it from
/root/reference and records its outputs so the tests can pin both the product
mesh module and the oracle's structured connectivity on a box without the
reference.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mesh_reference.npz")

CASES = [
    (1, [5]),
    (2, [4, 4]),
    (2, [3, 5]),
    (2, [16, 16]),
    (3, [2, 2, 2]),
    (3, [2, 3, 4]),
    (3, [4, 4, 4]),
]

BETAS = {
    1: [1.0],
    2: [1.0, -0.5],
    3: [0.2, 0.2, 0.2],
}


def main():
    sys.path.insert(0, REF)
    import ihdg.mesh as ref_mesh  # noqa: E402  (reference, read-only)

    out = {}
    ref1d = np.array([-1.0, -0.3, 0.45, 1.0])
    for ci, (dim, cells) in enumerate(CASES):
        m = ref_mesh.build_mesh(dim, cells)
        key = f"c{ci}"
        out[f"{key}_dim"] = np.array(dim)
        out[f"{key}_cells"] = np.array(cells)
        out[f"{key}_element_to_faces"] = m.element_to_faces
        out[f"{key}_neighbor_elements"] = m.neighbor_elements
        out[f"{key}_neighbor_faces"] = m.neighbor_faces
        out[f"{key}_face_axis"] = np.array([f.axis for f in m.faces])
        out[f"{key}_face_owner"] = np.array([f.owner for f in m.faces])
        out[f"{key}_face_neighbor"] = np.array([f.neighbor for f in m.faces])
        out[f"{key}_face_normal"] = np.array([f.normal for f in m.faces])
        out[f"{key}_face_centroid"] = np.array([f.centroid for f in m.faces])
        out[f"{key}_face_measure"] = np.array([f.measure for f in m.faces])
        out[f"{key}_face_points"] = np.array([m.face_points(f, ref1d[1:3]) for f in range(m.n_faces)])
        out[f"{key}_element_points"] = np.array(
            [m.element_points(e, [ref1d] * dim) for e in range(m.n_elements)])
        out[f"{key}_boundary_measure"] = np.array(m.boundary_surface_measure())
        b = np.array(BETAS[dim])
        tagged = ref_mesh.classify_boundary_faces(m, lambda x, b=b: np.tile(b, (x.shape[0], 1)))
        out[f"{key}_tags"] = np.array([f.tag for f in tagged.faces])
    out["ncases"] = np.array(len(CASES))
    out["ref1d"] = ref1d
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
