"""Multi-rank host logic on CPU (gloo): strip partition, ghost-layer halo
exchange and the rank-count independent norm reduction.

Each rank owns the layers [lb, le) of the slowest axis in a ghost-padded
buffer laid out exactly like the device buffers (one ghost layer before and
after), exchanges ghosts with ``paper_1711_01175_b200.partition.halo_exchange``
and sweeps its strip with the CPU oracle's local operators.  After several
sweeps the gathered strips must equal the single-process oracle sweep
bit-for-bit (block Jacobi is partition independent).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.ihdg_oracle import BOUNDARY, OracleProblem, OracleSolver
from paper_1711_01175_b200.partition import halo_exchange, strip_range  # noqa: F401

import scipy.linalg as sla


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _make_solver(kind, cells, periodic):
    d = len(cells)
    if kind == "cd":
        prob = OracleProblem("cd", d, beta=np.array([1.0, 0.6, 0.3][:d]), kappa=0.05)
        S = OracleSolver(prob, cells, 2, dt=0.02)
    elif kind == "sw":
        prob = OracleProblem("sw", 2, Phi=1.0, f_cor=1.0)
        S = OracleSolver(prob, cells, 2, periodic=periodic, dt=0.01)
    else:
        prob = OracleProblem("transport", d, beta=np.array([1.0, 0.5, 0.25][:d]))
        S = OracleSolver(prob, cells, 2)
        S.set_forcing(lambda x: np.sin(3 * x[:, 0]) + x[:, -1])
    return S


def _strip_sweep(S, buf, lb, le, ls, rhs_loc):
    """One sweep of the local strip reading neighbours from the padded buffer."""
    d = S.prob.dim
    nlay = le - lb
    out = np.empty((nlay * ls, S.nv))
    ncell_last = S.cells[-1]
    for el in range(nlay * ls):
        eg = lb * ls + el
        C = S.class_list[S.cls[eg]]
        r = rhs_loc[el].copy()
        for f in range(2 * d):
            nb = S.nbr[eg, f]
            if nb == BOUNDARY:
                continue
            lay = nb // ls
            if (f >> 1) == d - 1:  # neighbour across the layer axis -> maybe a ghost
                if f & 1:
                    lay_p = nlay + 1 if (lay < lb or lay >= le) else lay - lb + 1
                else:
                    lay_p = 0 if (lay < lb or lay >= le) else lay - lb + 1
            else:
                lay_p = lay - lb + 1
            src = buf[lay_p * ls + nb % ls]
            r += C["N"][f] @ src
        out[el] = sla.lu_solve((C["lu"], C["piv"]), r)
    return out


def _packed_exchange(buf, entries, ls, nlay, rank, world, per_last):
    """CPU mirror of DistributedSweeper._exchange: only the halo entries of
    the boundary layers cross the wire (packed), ghost rows hold nothing else."""
    from paper_1711_01175_b200.partition import halo_plan

    ops, recv = [], {}
    rows = {1: slice(ls, 2 * ls), 2: slice(nlay * ls, (nlay + 1) * ls),
            0: slice(0, ls), 3: slice((nlay + 1) * ls, (nlay + 2) * ls)}
    for peer, sdir, rdir, _ in halo_plan(rank, world, per_last):
        if entries[sdir]:
            layer = 1 if sdir == "to_lower" else 2
            ops.append(dist.P2POp(dist.isend, buf[rows[layer]][:, entries[sdir]].contiguous(), peer))
        if entries[rdir]:
            recv[rdir] = torch.zeros((ls, len(entries[rdir])), dtype=torch.float64)
            ops.append(dist.P2POp(dist.irecv, recv[rdir], peer))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for _, _, rdir, layer in halo_plan(rank, world, per_last):
        if entries[rdir]:
            g = buf[rows[layer]]
            g[:, entries[rdir]] = recv[rdir]


def _worker(rank, world, port, kind, cells, periodic, nsweeps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1711_01175_b200.partition import halo_entries, rows_sum_reference

        S = _make_solver(kind, cells, periodic)
        spec = _product_spec(kind, cells, periodic)
        entries = {dn: halo_entries(spec, dn) for dn in ("to_lower", "to_upper")}
        rng = np.random.default_rng(5)
        u0 = rng.normal(size=(S.nel, S.nv))
        rhs = S.rhs_static(u0 if S.dt is not None else None)
        ls = int(np.prod(cells[:-1]))
        lb, le = strip_range(cells[-1], rank, world)
        nlay = le - lb
        buf = torch.zeros(((nlay + 2) * ls, S.nv), dtype=torch.float64)
        buf[ls:(nlay + 1) * ls] = torch.from_numpy(u0[lb * ls:le * ls])
        rhs_loc = rhs[lb * ls:le * ls]
        per_last = bool(periodic and periodic[-1])
        for _ in range(nsweeps):
            _packed_exchange(buf, entries, ls, nlay, rank, world, per_last)
            new = _strip_sweep(S, buf.numpy(), lb, le, ls, rhs_loc)
            buf[ls:(nlay + 1) * ls] = torch.from_numpy(new)
        # tile partials: one per element here, rows = layers; the layer sums
        # of this rank go into its slice of a zeroed global array, all-reduced
        # (one non-zero term per layer: exact), then the fixed-order reduction
        part = (new ** 2).sum(axis=1).reshape(nlay, ls)
        layer_sums = torch.zeros(cells[-1], dtype=torch.float64)
        for i in range(nlay):
            rs = 0.0
            for x in part[i]:
                rs += float(x)
            layer_sums[lb + i] = rs
        dist.all_reduce(layer_sums)
        total = rows_sum_reference([[v] for v in layer_sums.tolist()])
        q.put((rank, lb, le, new, total))
    finally:
        dist.destroy_process_group()


def _product_spec(kind, cells, periodic):
    """The product's operator spec of the same problem (face weights -> halo entries)."""
    from paper_1711_01175_b200.assembly import build_spec
    from paper_1711_01175_b200.basis import build_operators
    from paper_1711_01175_b200.mesh import build_mesh
    from paper_1711_01175_b200.pde import ConvectionDiffusionProblem, ShallowWaterProblem, TransportProblem

    d = len(cells)
    mesh = build_mesh(d, cells, periodic=bool(periodic and periodic[-1]))
    ops = build_operators(2, d, mesh.h)
    if kind == "cd":
        return build_spec(mesh, ConvectionDiffusionProblem(kappa=0.05, beta=np.array([1.0, 0.6, 0.3][:d])), ops, 0.02)
    if kind == "sw":
        return build_spec(mesh, ShallowWaterProblem(Phi=1.0, f0=1.0), ops, 0.01)
    return build_spec(mesh, TransportProblem(beta=np.array([1.0, 0.5, 0.25][:d])), ops, None)


@pytest.mark.parametrize("kind,cells,periodic,world", [
    ("cd", [4, 6], None, 2),
    ("cd", [4, 7], None, 3),
    ("sw", [4, 6], [True, True], 2),
    ("sw", [3, 7], [True, True], 3),
    ("transport", [3, 2, 6], None, 3),
    ("transport", [3, 2, 5], None, 2),
])
def test_strip_partition_matches_single_process(kind, cells, periodic, world):
    nsweeps = 4
    S = _make_solver(kind, cells, periodic)
    rng = np.random.default_rng(5)
    u = rng.normal(size=(S.nel, S.nv))
    rhs = S.rhs_static(u if S.dt is not None else None)
    for _ in range(nsweeps):
        u = S.sweep(u, rhs)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, cells, periodic, nsweeps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_1711_01175_b200.partition import rows_sum_reference

    ls = int(np.prod(cells[:-1]))
    totals = set()
    for rank, lb, le, new, total in results:
        np.testing.assert_allclose(new, u[lb * ls:le * ls], rtol=1e-12, atol=1e-13)
        totals.add(total)
    # every rank derives the same norm (uneven strips included), equal to the
    # single-process two-level reduction (the strips' own rounding aside; the
    # device strips are bit-identical, tests/test_gpu_multirank.py)
    assert len(totals) == 1
    ref = rows_sum_reference((u ** 2).sum(axis=1).reshape(cells[-1], ls))
    assert abs(totals.pop() - ref) <= 1e-12 * abs(ref)


def test_strip_range():
    assert strip_range(10, 0, 3) == (0, 4)
    assert strip_range(10, 1, 3) == (4, 7)
    assert strip_range(10, 2, 3) == (7, 10)
    with pytest.raises(ValueError):
        strip_range(2, 0, 3)


@pytest.mark.parametrize("kind,cells,periodic", [("cd", [4, 6], None), ("sw", [4, 6], [True, True]),
                                                 ("transport", [3, 2, 6], None)])
def test_halo_entries_cover_the_coupling(kind, cells, periodic):
    """The packed halo carries every neighbour entry the local solve reads
    across the layer axis: with all other ghost entries zeroed, the oracle's
    neighbour coupling N_f gives the same result as with the full layer."""
    from paper_1711_01175_b200.partition import halo_entries

    S = _make_solver(kind, cells, periodic)
    spec = _product_spec(kind, cells, periodic)
    d = len(cells)
    rng = np.random.default_rng(2)
    full = rng.normal(size=S.nv)
    for direction, f in (("to_lower", 2 * (d - 1) + 1), ("to_upper", 2 * (d - 1))):
        ent = halo_entries(spec, direction)
        masked = np.zeros_like(full)
        masked[ent] = full[ent]
        for C in S.class_list:
            np.testing.assert_array_equal(C["N"][f] @ masked, C["N"][f] @ full)
        assert len(ent) < S.nv
