"""The N>1 host path on CPU with world_size-2 `gloo` (no GPU): the library's own
decomposition and face boxes (hfb_decomp_init / hfb_decomp_faces, pure host code in
libhfb.so) drive a halo exchange over torch.distributed; each rank advances its tile of
the diffusion program (diffusion.h90:23-41, numpy, same operation order, GLOBAL-index
boundaries) and the gathered result must equal the undecomposed oracle bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_1710_08616_b200 as hfb

NX, NY, NZ, STEPS, COEF, H = 23, 17, 9, 3, 0.1, 1


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def tile_step(a, d):
    """One diffuse_step on a tile array a[k, H+i-1, H+j-1] (halo ring of width H)."""
    out = a.copy()
    nx, ny = d.nx, d.ny
    gi = d.i0 + np.arange(1, nx + 1)
    gj = d.j0 + np.arange(1, ny + 1)
    c = a[:, H:H + nx, H:H + ny]
    s = np.empty_like(c)
    s[1:-1] = a[:-2, H:H + nx, H:H + ny] + a[2:, H:H + nx, H:H + ny]
    s[1:-1] = s[1:-1] + a[1:-1, H - 1:H - 1 + nx, H:H + ny]
    s[1:-1] = s[1:-1] + a[1:-1, H + 1:H + 1 + nx, H:H + ny]
    s[1:-1] = s[1:-1] + a[1:-1, H:H + nx, H - 1:H - 1 + ny]
    s[1:-1] = s[1:-1] + a[1:-1, H:H + nx, H + 1:H + 1 + ny]
    s[1:-1] = s[1:-1] - 6.0 * c[1:-1]
    new = c + COEF * s
    bnd = (gi[:, None] == 1) | (gi[:, None] == NX) | (gj[None, :] == 1) | (gj[None, :] == NY)
    bnd = np.broadcast_to(bnd, c.shape).copy()
    bnd[0] = True
    bnd[-1] = True
    out[:, H:H + nx, H:H + ny] = np.where(bnd, c, new)
    return out


def box_view(a, box):
    ilo, ihi, jlo, jhi = box
    return a[:, H + ilo - 1:H + ihi, H + jlo - 1:H + jhi]


def exchange(a, d):
    nbr = [d.west, d.east, d.south, d.north]
    for phase in (0, 1):
        reqs, recvs = [], []
        for side in (2 * phase, 2 * phase + 1):
            if nbr[side] < 0:
                continue
            send, recv = hfb.decomp_faces(d, side)
            buf = torch.from_numpy(np.ascontiguousarray(box_view(a, send)))
            rbuf = torch.empty(box_view(a, recv).shape, dtype=torch.float64)
            reqs.append(dist.isend(buf, nbr[side]))
            reqs.append(dist.irecv(rbuf, nbr[side]))
            recvs.append((recv, rbuf))
        for r in reqs:
            r.wait()
        for recv, rbuf in recvs:
            box_view(a, recv)[...] = rbuf.numpy()


def worker(rank, world, port, px, py, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = hfb.decomp_init(NX, NY, NZ, px, py, rank, halo=H)
    g = oracle.fill((NZ, NX, NY), 1, 280.0, 10.0)
    a = np.zeros((NZ, d.nx + 2 * H, d.ny + 2 * H))
    a[:, H:H + d.nx, H:H + d.ny] = g[:, d.i0:d.i0 + d.nx, d.j0:d.j0 + d.ny]
    for _ in range(STEPS):
        exchange(a, d)
        a = tile_step(a, d)
    q.put((rank, int(d.i0), int(d.j0), a[:, H:H + d.nx, H:H + d.ny].copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("px,py", [(2, 1), (1, 2)])
def test_gloo_two_rank_diffusion_equals_oracle(px, py):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, px, py, q)) for r in range(2)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out = np.empty((NZ, NX, NY))
    for _, i0, j0, t in parts:
        out[:, i0:i0 + t.shape[1], j0:j0 + t.shape[2]] = t
    ref_old = oracle.fill((NZ, NX, NY), 1, 280.0, 10.0)
    ref_new = np.zeros_like(ref_old)
    oracle.diffusion_run(STEPS, COEF, ref_old, ref_new)
    assert np.array_equal(out.view(np.uint64), ref_old.view(np.uint64))
