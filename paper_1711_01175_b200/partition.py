"""Strip partition of the mesh across ranks + per-sweep halo exchange.

SURVEY.md 8e: block-Jacobi with a one-iteration lag is partition independent
(PAPER.md:328-342), so each rank owns a contiguous range of element layers of
the slowest axis (y-rows in 2D, z-planes in 3D; contiguous element ranges in
the lexicographic numbering, mesh.py:73-75) and, before every sweep, receives
the neighbouring ranks' boundary layers of iterate k into its ghost layers.
The stopping norm is made rank-count independent by all-gathering the
per-tile partials and reducing them in global tile order on every rank.

The functions here operate on torch tensors of any device: NCCL over NVLink
on the B200 box, gloo on CPU in the tests (tests/test_partition_gloo.py).
"""

from __future__ import annotations

__all__ = ["strip_range", "halo_exchange", "halo_ops"]


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


def halo_ops(rank: int, world: int, periodic: bool):
    """(send_to_lower, recv_from_lower, send_to_upper, recv_from_upper) peer
    ranks or None.  Rank r's first local layer is the ghost_hi of rank r-1,
    its last local layer the ghost_lo of rank r+1."""
    lower = rank - 1 if rank > 0 else (world - 1 if periodic else None)
    upper = rank + 1 if rank < world - 1 else (0 if periodic else None)
    return lower, upper


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
