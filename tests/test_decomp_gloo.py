"""The N>1 host path on CPU with `gloo` (no GPU): each rank holds its tile in the engine's
DEVICE layout (hfb_layout_of: I fastest, padded rows, 2-cell halo ring) and exchanges halos
exactly as the NCCL transport does (hfb_runtime.cu nccl halo exchange: two phases, west/east
then south/north so corners travel), with the library's own pieces — the decomposition
(hfb_decomp_init), the face boxes (hfb_decomp_faces) and the host twins of the pack /
unpack kernels (hfb_pack_box_host / hfb_unpack_box_host: the kernels' element order) —
over torch.distributed send/recv. Each rank advances its tile with the diffusion step
(diffusion.h90:23-41 in the reference's operation order, GLOBAL-index boundaries; the one
piece of test arithmetic, since the kernels need a GPU); the gathered result must equal
the undecomposed oracle bit for bit. Ranks: 2 (both splits) and 4 (2 x 2: corners)."""
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


def tile_step(t, d):
    """One diffuse_step on the tile's padded view a[k, j', i'] (halo width H)."""
    a = t.padded(H)
    nx, ny = d.nx, d.ny
    gi = d.i0 + np.arange(1, nx + 1)
    gj = d.j0 + np.arange(1, ny + 1)
    c = a[:, H:H + ny, H:H + nx]
    s = np.empty_like(c)
    s[1:-1] = a[:-2, H:H + ny, H:H + nx] + a[2:, H:H + ny, H:H + nx]
    s[1:-1] = s[1:-1] + a[1:-1, H:H + ny, H - 1:H - 1 + nx]
    s[1:-1] = s[1:-1] + a[1:-1, H:H + ny, H + 1:H + 1 + nx]
    s[1:-1] = s[1:-1] + a[1:-1, H - 1:H - 1 + ny, H:H + nx]
    s[1:-1] = s[1:-1] + a[1:-1, H + 1:H + 1 + ny, H:H + nx]
    s[1:-1] = s[1:-1] - 6.0 * c[1:-1]
    new = c + COEF * s
    bnd = (gj[:, None] == 1) | (gj[:, None] == NY) | (gi[None, :] == 1) | (gi[None, :] == NX)
    bnd = np.broadcast_to(bnd, c.shape).copy()
    bnd[0] = True
    bnd[-1] = True
    t.interior()[...] = np.where(bnd, c, new)


def exchange(t, d):
    """The NCCL transport's two-phase halo exchange with gloo point-to-point messages."""
    nbr = [d.west, d.east, d.south, d.north]
    for phase in (0, 1):
        reqs, recvs = [], []
        for side in (2 * phase, 2 * phase + 1):
            if nbr[side] < 0:
                continue
            send, recv = hfb.decomp_faces(d, side)
            buf = torch.from_numpy(t.pack(send))
            n = (recv[1] - recv[0] + 1) * (recv[3] - recv[2] + 1) * t.nk
            rbuf = torch.empty(n, dtype=torch.float64)
            reqs.append(dist.isend(buf, nbr[side]))
            reqs.append(dist.irecv(rbuf, nbr[side]))
            recvs.append((recv, rbuf))
        for r in reqs:
            r.wait()
        for recv, rbuf in recvs:
            t.unpack(recv, rbuf.numpy())


def worker(rank, world, port, px, py, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = hfb.decomp_init(NX, NY, NZ, px, py, rank, halo=H)
    g = oracle.fill((NZ, NX, NY), 1, 280.0, 10.0)
    t = hfb.TileLayout(int(d.nx), int(d.ny), NZ)
    t.interior()[...] = g[:, d.i0:d.i0 + d.nx, d.j0:d.j0 + d.ny].transpose(0, 2, 1)
    for _ in range(STEPS):
        exchange(t, d)
        tile_step(t, d)
    q.put((rank, int(d.i0), int(d.j0), t.interior().transpose(0, 2, 1).copy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("px,py", [(2, 1), (1, 2), (2, 2)])
def test_gloo_ranks_diffusion_equals_oracle(px, py):
    world = px * py
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, px, py, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=120) for _ in range(world)]
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


def test_pack_box_host_element_order():
    """The host twin packs i fastest, then j, then k (the kernels' order) and unpack
    inverts it, halo-ring coordinates included."""
    t = hfb.TileLayout(5, 4, 3)
    t.buf[:] = np.arange(t.alloc, dtype=np.float64)
    a = t.padded(2)
    box = (0, 2, -1, 1)  # i 0..2, j -1..1: halo ring cells included
    got = t.pack(box)
    want = np.concatenate([a[k, 2 + box[2] - 1:2 + box[3], 2 + box[0] - 1:2 + box[1]].ravel()
                           for k in range(3)])
    assert np.array_equal(got, want)
    t.unpack(box, -got)
    assert np.array_equal(t.pack(box), -got)
