"""Strip partition of the mesh across ranks + per-sweep halo exchange.

SURVEY.md 8e: block-Jacobi with a one-iteration lag is partition independent
(PAPER.md:328-342), so each rank owns a contiguous range of element layers of
the slowest axis (y-rows in 2D, z-planes in 3D; contiguous element ranges in
the lexicographic numbering, mesh.py:73-75) and, before every sweep, receives
the neighbouring ranks' boundary data of iterate k into its ghost layers.
Only the face-node entries the neighbour's sweep reads cross the wire
(``halo_entries``: the components with a nonzero neighbour face weight at the
nodes of the shared face -- 2 x 7 doubles per element at config 5 instead of
147), packed and unpacked on the device (ihdg_halo_pack / _unpack).
The stopping norm is made rank-count independent by reducing each element
layer's tile partials on its owner (ihdg_layer_sums), all-reducing the layer
sums (every layer has exactly one non-zero contribution, so the sum is exact)
and reducing them in a fixed order on every rank (ihdg_finalize, the order of
the fused single-rank finalize).

The functions here operate on torch tensors of any device: NCCL over NVLink
on the B200 box, gloo on CPU in the tests (tests/test_partition_gloo.py).
"""

from __future__ import annotations

__all__ = ["strip_range", "halo_exchange", "halo_ops", "halo_entries", "face_node_vidx", "halo_plan",
           "rows_sum_reference"]


def strip_range(n_layers: int, rank: int, world: int) -> tuple[int, int]:
    """Layers [begin, end) of ``rank``: an even split, the remainder spread
    over the first ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if n_layers < world:
        raise ValueError(f"{n_layers} layers cannot be split over {world} ranks")
    base, rem = divmod(n_layers, world)
    begin = rank * base + min(rank, rem)
    return begin, begin + base + (1 if rank < rem else 0)


def face_node_vidx(dim: int, n1: int, f: int, n: int) -> int:
    """Volume node of node n of local face f (tangential axes increasing, the
    smallest fastest; nodes lexicographic, axis 0 fastest: mesh.py:155-187)."""
    a, s = divmod(f, 2)
    v, mul = 0, 1
    for b in range(dim):
        if b == a:
            ib = n1 - 1 if s else 0
        else:
            ib = n % n1
            n //= n1
        v += ib * mul
        mul *= n1
    return v


def halo_entries(spec, direction: str) -> list:
    """Element-local DOF entries (component * (p+1)^d + node) of a boundary
    layer that a neighbouring rank's sweep reads: direction "to_lower" (my
    first layer -> the lower rank's ghost_hi, read across its high face of
    the layer axis) or "to_upper" (my last layer -> the upper rank's
    ghost_lo).  The neighbour face scalar of face f is
    q = sum_c face_w[f][c] u_nbr[c][face f^1 node] (csrc/ihdg_ws.cuh,
    ihdg_kernels.cuh), so only components with a nonzero face weight at the
    nodes of the shared face are needed."""
    d, n1 = spec.dim, spec.n1
    f_recv = 2 * (d - 1) + (1 if direction == "to_lower" else 0)
    if direction not in ("to_lower", "to_upper"):
        raise ValueError(direction)
    if not spec.coupled[f_recv]:
        return []
    nf = n1 ** (d - 1)
    npn = n1 ** d
    comps = [c for c in range(spec.ncomp) if float(spec.face_w[f_recv, c]) != 0.0]
    return [c * npn + face_node_vidx(d, n1, f_recv ^ 1, n) for c in comps for n in range(nf)]


def halo_ops(rank: int, world: int, periodic: bool):
    """(send_to_lower, recv_from_lower, send_to_upper, recv_from_upper) peer
    ranks or None.  Rank r's first local layer is the ghost_hi of rank r-1,
    its last local layer the ghost_lo of rank r+1."""
    lower = rank - 1 if rank > 0 else (world - 1 if periodic else None)
    upper = rank + 1 if rank < world - 1 else (0 if periodic else None)
    return lower, upper


def halo_plan(rank: int, world: int, periodic: bool) -> list:
    """Ordered P2P plan of one halo exchange: (peer, send entries, receive
    entries, ghost row to unpack into: 0 = ghost_lo, 3 = ghost_hi).  My first
    layer goes to the lower rank ("to_lower" entries), my last to the upper
    rank ("to_upper"); the lower rank's last layer arrives in ghost_lo, the
    upper rank's first in ghost_hi.  At world = 2 with a periodic layer axis
    both neighbours are one peer and messages of a pair of ranks match in
    issue order, so rank 1 issues its plan reversed."""
    lower, upper = halo_ops(rank, world, periodic)
    plan = []
    if lower is not None:
        plan.append((lower, "to_lower", "to_upper", 0))
    if upper is not None:
        plan.append((upper, "to_upper", "to_lower", 3))
    if world == 2 and periodic and rank == 1:
        plan = plan[::-1]
    return plan


def rows_sum_reference(rows) -> float:
    """Host restatement of the device's fixed-order norm reduction
    (csrc/ihdg_kernels.cuh rows_sum): every row summed sequentially, virtual
    lane v of 256 sums rows v, v+256, ... in order, then a fixed binary tree."""
    red = [0.0] * 256
    for v in range(256):
        s = 0.0
        for r in range(v, len(rows), 256):
            rs = 0.0
            for x in rows[r]:
                rs += float(x)
            s += rs
        red[v] = s
    w = 128
    while w > 0:
        for v in range(w):
            red[v] += red[v + w]
        w >>= 1
    return red[0]


def halo_exchange(buf, layer_elems: int, n_local_layers: int, rank: int, world: int,
                  periodic: bool, group=None, host_staging: bool = False) -> None:
    """Fill the ghost layers of the ghost-padded state ``buf``
    [(n_local_layers + 2) * layer_elems, NV] from the neighbouring ranks.

    Layout: rows [0, L) ghost_lo | [L, L + nL) local | [L + nL, 2L + nL) ghost_hi
    with L = layer_elems elements per layer.
    """
    import torch.distributed as dist

    if world == 1:
        return
    L, nL = layer_elems, n_local_layers
    if host_staging and buf.is_cuda:
        # gloo path for device buffers: exchange host copies of the boundary
        # layers (test mode on a single GPU; no kernel waits on another rank)
        stage = buf.new_zeros(((nL + 2) * L,) + tuple(buf.shape[1:]), device="cpu")
        stage[L: 2 * L] = buf[L: 2 * L].cpu()
        stage[nL * L: (nL + 1) * L] = buf[nL * L: (nL + 1) * L].cpu()
        halo_exchange(stage, L, nL, rank, world, periodic, group)
        lower, upper = halo_ops(rank, world, periodic)
        if lower is not None:
            buf[0: L].copy_(stage[0: L])
        if upper is not None:
            buf[(nL + 1) * L: (nL + 2) * L].copy_(stage[(nL + 1) * L: (nL + 2) * L])
        return
    first = buf[L: 2 * L]
    last = buf[nL * L: (nL + 1) * L]
    ghost_lo = buf[0: L]
    ghost_hi = buf[(nL + 1) * L: (nL + 2) * L]
    lower, upper = halo_ops(rank, world, periodic)
    ops = []
    if world == 2 and periodic:
        # both neighbours are the same peer; messages between one pair of
        # ranks match in issue order per direction, so rank 1 sends its last
        # layer (rank 0's ghost_lo) first and receives into ghost_hi first.
        peer = 1 - rank
        if rank == 0:
            seq = [(dist.isend, first), (dist.irecv, ghost_lo), (dist.isend, last), (dist.irecv, ghost_hi)]
        else:
            seq = [(dist.isend, last), (dist.irecv, ghost_hi), (dist.isend, first), (dist.irecv, ghost_lo)]
        ops = [dist.P2POp(fn, t, peer, group) for fn, t in seq]
    else:
        if lower is not None:
            ops.append(dist.P2POp(dist.isend, first, lower, group))
            ops.append(dist.P2POp(dist.irecv, ghost_lo, lower, group))
        if upper is not None:
            ops.append(dist.P2POp(dist.isend, last, upper, group))
            ops.append(dist.P2POp(dist.irecv, ghost_hi, upper, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
