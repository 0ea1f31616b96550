"""The code paths that only run with one GPU PER RANK (skipped on boxes with fewer than
two GPUs; the driver's multi-GPU box runs them):

  * the NCCL transport (hfb_set_decomposition with an ncclUniqueId: pack -> grouped
    ncclSend/ncclRecv -> unpack, two phases; ncclAllReduce for the reduction), which NCCL
    refuses to run with two ranks on one device;
  * the peer transport across devices: CUDA IPC handles opened on another GPU
    (cudaIpcMemLazyEnablePeerAccess), halo pushes and the fused epilogue stores going over
    NVLink, release/acquire flags at system scope between devices, graph replay;
  * bench.py's multi-GPU line (torchrun, one rank per GPU, NCCL process group).

Every decomposed result must equal the undecomposed oracle bit for bit (1e-12 for the
tree-summed reduction)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1710_08616_b200 as hfb
from cases import APPS, DYCORE_FILLS, DYCORE_SCALARS, PHYS_FILLS, PHYS_SCALARS, Case, _asu
from golden_io import bits_equal, decl, make_inputs, run_oracle
from test_gpu_decomp import global_extent, tile_ints, tile_slices

NDEV = torch.cuda.device_count() if torch.cuda.is_available() else 0
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(NDEV < 2, reason="needs one GPU per rank (>= 2 GPUs)")]
ROOT = Path(__file__).resolve().parents[1]

CASES = {
    "dycore": Case("m_dycore", "dycore", dict(nx=70, ny=45, nz=20, nsteps=4),
                   dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    "dycore_full": Case("m_full", "dycore_full", dict(nx=70, ny=45, nz=20, nsteps=2),
                        dict(DYCORE_SCALARS, **PHYS_SCALARS), dict(DYCORE_FILLS, **PHYS_FILLS)),
    "diffusion": Case("m_diff", "diffusion", dict(nx=40, ny=36, nz=12, nsteps=3),
                      dict(coef=0.1), {"t_old": (1, 280.0, 10.0)}, unset=["t_new"]),
    "reduction": Case("m_red", "reduction", dict(nx=67, ny=45, nz=20), dict(total=0.0),
                      {"y": (6, 0.0, 1.0)}),
    "asuca": _asu("m_asuca", 70, 45, 20, 1, nbnd=3),
}
HALO = {"dycore": 2, "dycore_full": 2, "diffusion": 1, "reduction": 0, "asuca": 2}


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, name, px, py, transport, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = CASES[name]
        garr = make_inputs(case)
        gnx, gny = global_extent(case)
        d = hfb.decomp_init(gnx, gny, case.ints.get("nz", 1), px, py, rank, halo=HALO[name])
        eng = hfb.Engine(APPS[case.app].prog, device=rank)
        if transport == "nccl":
            obj = [hfb.runtime.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            eng.set_decomposition(d, obj[0])
        else:
            eng.set_decomposition(d)
        ints = tile_ints(case, d)
        for k, v in ints.items():
            eng.set(k, int(v))
        for k, v in case.reals.items():
            eng.set(k, float(v))
        tiles = {}
        for n, a in garr.items():
            tiles[n] = np.ascontiguousarray(a[tile_slices(case.app, n, a, d)])
            _, lower = decl(case.app, n, ints)
            eng.bind(n, tiles[n], lower=lower)
        if transport == "peer":
            eng.attach_peers()
        if mode == "graph":
            step = "full_step" if case.app == "dycore_full" else "dycore_step"
            for n in tiles:
                eng.copy_to_device(n)
            for _ in range(case.ints["nsteps"] // 2):
                eng.run_graph(step, 2)
            for n in tiles:
                eng.copy_from_device(n)
        else:
            eng.run(APPS[case.app].entry)
        total = eng.get("total") if case.app == "reduction" else None
        q.put((rank, tiles, total, eng.halo_bytes(), None))
        dist.barrier()
        eng.close()
    except Exception as e:
        q.put((rank, None, None, 0, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def run(name, px, py, transport, mode="main"):
    world = px * py
    if world > NDEV:
        pytest.skip(f"needs {world} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, name, px, py, transport, mode, q))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        parts = [q.get(timeout=300) for _ in range(world)]
        for p in procs:
            p.join(timeout=120)
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
    errors = [e for *_, e in parts if e]
    assert not errors, errors
    case = CASES[name]
    garr = make_inputs(case)
    ref = {k: v.copy() for k, v in garr.items()}
    res = run_oracle(case, ref)
    if case.app == "reduction":
        for _, _, total, _, _ in parts:
            assert abs(total - res["total"]) <= 1e-12 * abs(res["total"])
        return parts
    gnx, gny = global_extent(case)
    out = {k: np.empty_like(v) for k, v in garr.items()}
    for rank, tiles, _, _, _ in parts:
        d = hfb.decomp_init(gnx, gny, case.ints.get("nz", 1), px, py, rank, halo=HALO[name])
        for k, t in tiles.items():
            out[k][tile_slices(case.app, k, out[k], d)] = t
    names = ("t_old", "t_new") if case.app == "diffusion" else APPS[case.app].outputs
    for k in names:
        assert bits_equal(out[k], ref[k]), f"{name} {transport} {px}x{py}: {k} differs"
    assert all(p[3] > 0 for p in parts)
    return parts


@pytest.mark.parametrize("name", ["dycore", "dycore_full", "diffusion", "reduction", "asuca"])
def test_nccl_transport_two_gpus(name):
    run(name, 2, 1, "nccl")


@pytest.mark.parametrize("name", ["dycore", "diffusion", "reduction", "asuca"])
def test_peer_transport_across_devices(name):
    run(name, 2, 1, "peer")


def test_peer_transport_graph_replay_across_devices():
    run("dycore", 2, 1, "peer", mode="graph")


def test_four_gpus_2x2_both_transports():
    for transport in ("nccl", "peer"):
        run("dycore", 2, 2, transport)


def test_bench_multi_gpu_line():
    """bench.py --gpus 2 under torchrun (NCCL process group, one rank per GPU): one JSON
    line with the whole-job value and the halo traffic."""
    env = {k: v for k, v in os.environ.items() if not k.startswith("HFB_")}
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(free_port()), str(ROOT / "bench.py"), "--gpus", "2", "--steps", "4",
                        "--warmup", "3", "--tile512", "--no-secondary"],
                       capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["halo"]["bytes_per_step_rank0"] > 0
