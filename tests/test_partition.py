"""Element partition on the CPU.

* The library's host-only partition arithmetic (hbpdc_partition) covers the
  mesh exactly once and its neighbour relation is symmetric.
* world_size-2 gloo runs: each rank takes its block from hbpdc_partition,
  exchanges face traces with the halo convention of comm.h (send side s to
  nbr[s]; slot s <- nbr[s]'s side s ^ 1) over torch.distributed, and
  evaluates the oracle's R^(1) on its block padded with those ghost traces.
  The assembled blocks equal the oracle's global R^(1) (the same property
  the GPU loopback / NCCL tests check for the CUDA path).
"""
import os
import socket

import numpy as np
import pytest

from oracle import basis, dgsem, physics
from paper_2109_04804_b200 import hbpdc, inputs


@pytest.mark.parametrize("dim,nx,ny,px,py", [(2, 8, 6, 2, 3), (2, 8, 8, 4, 2), (2, 4, 4, 1, 1),
                                             (1, 12, 1, 3, 1), (2, 6, 4, 6, 1)])
def test_partition_covers_mesh_and_is_symmetric(dim, nx, ny, px, py):
    owner = -np.ones((ny, nx), int)
    nbrs = {}
    for r in range(px * py):
        ex0, ey0, nxl, nyl, nb = hbpdc.partition(dim, nx, ny, px, py, r)
        assert nxl == nx // px and nyl == ny // py
        assert (owner[ey0:ey0 + nyl, ex0:ex0 + nxl] == -1).all()
        owner[ey0:ey0 + nyl, ex0:ex0 + nxl] = r
        nbrs[r] = nb
    assert (owner >= 0).all()
    for r, nb in nbrs.items():
        for s in range(4 if dim == 2 else 2):
            assert nbrs[nb[s]][s ^ 1] == r          # my +x neighbour has me as its -x neighbour


def test_partition_rejects_non_dividing_grid():
    with pytest.raises(hbpdc.HbpdcError):
        hbpdc.partition(2, 10, 8, 3, 2, 0)


# ---------------------------------------------------------------------------------
# gloo: halo convention + oracle R1 on padded blocks

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _global_state(kind, N, nx, ny):
    eq = physics.Equation(kind, a=(1.0, -0.6))
    d = dgsem.Disc(basis.build_basis(N, "gll"), dgsem.Mesh(2, nx, ny, 0.0, 1.0, 0.0, 1.0), eq)
    X, Y = d.node_coords()
    if kind == "advection":
        W = inputs.initial_state("C2", (X, Y))
    else:
        W = inputs.initial_state("C4", (X, Y))
    W = inputs.perturbed_state(W, inputs.MASTER_SEED + 77)
    return d, W


def _worker(rank, world, port, kind, N, nx, ny, px, py, q):
    import torch.distributed as dist
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        d, W = _global_state(kind, N, nx, ny)
        p, nv = d.p, d.nv
        Wf = W.reshape(ny, nx, nv, p, p)
        ex0, ey0, nxl, nyl, nb = hbpdc.partition(2, nx, ny, px, py, rank)
        loc = Wf[ey0:ey0 + nyl, ex0:ex0 + nxl].copy()
        hx, hy = px > 1, py > 1
        # own face traces per side (GLL: boundary nodes): (count along side, nv, p)
        faces = {0: loc[:, 0, :, :, 0], 1: loc[:, -1, :, :, -1], 2: loc[0, :, :, 0, :], 3: loc[-1, :, :, -1, :]}
        active = [hx, hx, hy, hy]
        reqs, recv = [], {}
        for s in range(4):
            if active[s]:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(faces[s])), dst=nb[s], tag=s))
        for s in range(4):
            if active[s]:
                buf = torch.empty(faces[s ^ 1].shape, dtype=torch.float64)
                reqs.append(dist.irecv(buf, src=nb[s], tag=s ^ 1))
                recv[s] = buf
        for r in reqs:
            r.wait()
        # padded block: ghost ring on the split directions, zero except face nodes
        ox, oy = int(hx), int(hy)
        ext = np.zeros((nyl + 2 * oy, nxl + 2 * ox, nv, p, p))
        ext[oy:oy + nyl, ox:ox + nxl] = loc
        if hx:
            ext[oy:oy + nyl, 0, :, :, -1] = recv[0].numpy()      # west ghost: its +x face
            ext[oy:oy + nyl, -1, :, :, 0] = recv[1].numpy()      # east ghost: its -x face
        if hy:
            ext[0, ox:ox + nxl, :, -1, :] = recv[2].numpy()
            ext[-1, ox:ox + nxl, :, 0, :] = recv[3].numpy()
        me = d.mesh
        dx, dy = me.dx, me.dy
        de = dgsem.Disc(d.basis, dgsem.Mesh(2, nxl + 2 * ox, nyl + 2 * oy, 0.0, dx * (nxl + 2 * ox),
                                            0.0, dy * (nyl + 2 * oy)), d.eq)
        R = dgsem.rhs1(de, ext.reshape(-1)).reshape(ext.shape)[oy:oy + nyl, ox:ox + nxl]
        q.put((rank, ex0, ey0, R))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,px,py", [("euler", 2, 1), ("euler", 1, 2), ("advection", 2, 1)])
def test_gloo_halo_convention_reproduces_global_r1(kind, px, py):
    import torch.multiprocessing as mp
    N, nx, ny = 3, 4, 4
    world = px * py
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, N, nx, ny, px, py, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    d, W = _global_state(kind, N, nx, ny)
    Rg = dgsem.rhs1(d, W).reshape(ny, nx, d.nv, d.p, d.p)
    for rank, ex0, ey0, R in out:
        blk = Rg[ey0:ey0 + R.shape[0], ex0:ex0 + R.shape[1]]
        err = np.linalg.norm(R - blk) / np.linalg.norm(blk)
        assert err <= 1e-13, (rank, err)
