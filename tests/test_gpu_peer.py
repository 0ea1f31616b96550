"""The peer-memory transport (hfb_peer_export / hfb_peer_attach): one PROCESS per rank,
the ranks' device buffers mapped into each other by CUDA IPC, halos stored straight into
the neighbours' halo rings by one push kernel (corners to the diagonal neighbours) with a
release/acquire flag per neighbour, reductions summed in rank order through peer memory.
On a multi-GPU node the stores travel over NVLink/NVSwitch; here every rank's process
shares the one GPU (CUDA IPC works within a device, NCCL refuses duplicate GPUs), which
exercises the same kernels, flags and handle plumbing. The assembled tiles must equal
the undecomposed oracle bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1710_08616_b200 as hfb
from cases import APPS, DYCORE_FILLS, DYCORE_SCALARS, PHYS_FILLS, PHYS_SCALARS, Case, _asu
from golden_io import bits_equal, decl, make_inputs, run_oracle
from test_gpu_decomp import global_extent, tile_ints, tile_slices

pytestmark = pytest.mark.gpu

PEER_CASES = {
    "dycore": Case("p_dycore", "dycore", dict(nx=70, ny=45, nz=20, nsteps=3),
                   dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    "dycore4": Case("p_dycore4", "dycore", dict(nx=70, ny=45, nz=20, nsteps=4),
                    dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    "dycore_full4": Case("p_full4", "dycore_full", dict(nx=70, ny=45, nz=20, nsteps=4),
                         dict(DYCORE_SCALARS, **PHYS_SCALARS), dict(DYCORE_FILLS, **PHYS_FILLS)),
    "dycore_full": Case("p_full", "dycore_full", dict(nx=70, ny=45, nz=20, nsteps=2),
                        dict(DYCORE_SCALARS, **PHYS_SCALARS),
                        dict(DYCORE_FILLS, **PHYS_FILLS)),
    "dycore_rk3": Case("p_rk3", "dycore_rk3", dict(nx=70, ny=45, nz=20, nsteps=2),
                       dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    # the ASUCA scheme: 28 exchanges per step (stage state, fu/fv, p/u/v, pa), nbnd = 3
    # damping band across the tile edges; 2 short steps in stage 1 (nsound = 6)
    "asuca": _asu("p_asuca", 70, 45, 20, 2, nbnd=3),
    # tiles wide enough for whole-tile boundary strips (32 columns, 4 rows) in both
    # directions when the exchange is overlapped
    "asuca_wide": _asu("p_asuca_w", 150, 30, 12, 1, nbnd=3),
    "dycore_wide": Case("p_dyn_w", "dycore", dict(nx=150, ny=30, nz=20, nsteps=3),
                        dict(DYCORE_SCALARS), dict(DYCORE_FILLS)),
    "diffusion": Case("p_diff", "diffusion", dict(nx=40, ny=36, nz=12, nsteps=3),
                      dict(coef=0.1), {"t_old": (1, 280.0, 10.0)}, unset=["t_new"]),
    "bounded": Case("p_bnd", "bounded", dict(nx=37, ny=21), {},
                    {"a": (4, 0.0, 1.0), "b": (6, -1.0, 0.5)}),
    "damping": Case("p_damp", "damping",
                    dict(nx_mn=-1, nx_mx=35, ny_mn=0, ny_mx=20, nz_mn=1, nz_mx=9),
                    dict(tratio_bnd=0.3, mtratio_bnd=0.7),
                    {"dens_ref_f": (2, 1.0, 1.0), "dens_ptb_bnd": (3, -0.005, 0.01)}),
    "reduction": Case("p_red", "reduction", dict(nx=67, ny=45, nz=20), dict(total=0.0),
                      {"y": (6, 0.0, 1.0)}),
}
HALO = {"asuca": 2, "asuca_wide": 2, "dycore_wide": 2, "dycore": 2, "dycore4": 2, "dycore_full4": 2, "dycore_full": 2, "dycore_rk3": 2, "diffusion": 1, "reduction": 0,
        "bounded": 1, "damping": 0}


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, name, px, py, q, per_step=False, ordered=False, options=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = PEER_CASES[name]
        garr = make_inputs(case)
        gnx, gny = global_extent(case)
        d = hfb.decomp_init(gnx, gny, case.ints.get("nz", 1), px, py, rank, halo=HALO[name])
        eng = hfb.Engine(APPS[case.app].prog, device=0)
        eng.set_decomposition(d)
        for k, v in (options or {}).items():
            eng.set_option(k, v)
        if ordered:
            eng.set_reduction_order(True)
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
        eng.attach_peers()
        if per_step:  # the bench's device-resident path: copy-in, n steps, copy-out
            step = {"dycore_full": "full_step", "asuca": "asuca_step"}.get(case.app,
                                                                          "dycore_step")
            for n in tiles:
                eng.copy_to_device(n)
            if per_step == "graph":  # CUDA graphs of 2 steps, replayed
                for _ in range(case.ints["nsteps"] // 2):
                    stats = eng.run_graph(step, 2)
            else:
                for _ in range(case.ints["nsteps"]):
                    stats = eng.enqueue(step)
            eng.synchronize()
            for n in tiles:
                eng.copy_from_device(n)
        else:
            stats = eng.run(APPS[case.app].entry)
        total = eng.get("total") if case.app == "reduction" else None
        q.put((rank, eng.peer_stats(), tiles, total,
               eng.halo_bytes(), stats.native_launches, None))
        dist.barrier()
        eng.close()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, None, None, None, 0, 0, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def run_peer(name, px, py, per_step=False, ordered=False, options=None):
    world = px * py
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, name, px, py, q, per_step, ordered, options))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        parts = [q.get(timeout=300) for _ in range(world)]
        for p in procs:
            p.join(timeout=120)
    finally:
        for p in procs:  # a hung rank (e.g. a flag never released) must not outlive the test
            if p.is_alive():
                p.kill()
    errors = [e for *_, e in parts if e]
    assert not errors, errors
    for p in procs:
        assert p.exitcode == 0
    case = PEER_CASES[name]
    garr = make_inputs(case)
    out = {k: np.empty_like(v) for k, v in garr.items()}
    gnx, gny = global_extent(case)
    for rank, _, tiles, _, _, _, _ in parts:
        d = hfb.decomp_init(gnx, gny, case.ints.get("nz", 1), px, py, rank, halo=HALO[name])
        for k, t in tiles.items():
            out[k][tile_slices(case.app, k, out[k], d)] = t
    return case, garr, out, parts


@pytest.mark.parametrize("name,px,py", [("dycore", 2, 1), ("dycore", 2, 2), ("dycore", 4, 2),
                                        ("dycore_full", 2, 2), ("dycore_rk3", 2, 2),
                                        ("diffusion", 2, 2), ("dycore", 3, 2),
                                        ("bounded", 2, 3), ("damping", 2, 2)])
def test_peer_transport_equals_single_domain(name, px, py):
    case, garr, out, parts = run_peer(name, px, py)
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    names = {"diffusion": ("t_old", "t_new"), "damping": ("dens_ptb_damp",)}.get(
        case.app, APPS[case.app].outputs)
    for k in names:
        assert bits_equal(out[k], ref[k]), f"{name} {px}x{py}: {k} differs"
    if HALO[name] == 0:  # pointwise: no exchange at all
        assert all(p[1] == (0, 0) and p[4] == 0 for p in parts)
        return
    assert all(p[4] > 0 for p in parts)  # every rank moved halo bytes
    n = case.ints.get("nsteps", 1)
    # dycore: the first step after the copy-in pushes, the next ones are handed off by the
    # previous step's epilogue; diffusion pushes every step
    want = ((3 * n, 0) if case.app == "dycore_rk3"  # RK stages push (3 per step)
            else (1, n - 1) if case.app.startswith("dycore") else (n, 0))
    assert all(p[1] == want for p in parts), [p[1] for p in parts]


def test_peer_reduction_is_rank_ordered_and_identical_everywhere():
    case, garr, _, parts = run_peer("reduction", 2, 2)
    totals = [p[3] for p in parts]
    assert len({np.float64(t).view(np.uint64) for t in totals}) == 1
    ref = run_oracle(case, {k: v.copy() for k, v in garr.items()})["total"]
    assert abs(totals[0] - ref) <= 1e-12 * abs(ref)


@pytest.mark.parametrize("name,overlap", [("dycore", True), ("dycore", False),
                                           ("dycore_wide", True)])
def test_peer_fused_halo_hand_off_per_step_entries(name, overlap):
    """Consecutive dycore_step entries hand the halos over in the step kernel's epilogue
    (boundary strips store into the neighbours' next-step halo rings; the next exchange
    only waits for their flags). Without overlap the single full-span launch carries the
    remote epilogue. Both equal the undecomposed oracle bit for bit."""
    case, garr, out, parts = run_peer(name, 2, 2, per_step=True,
                                      options={"overlap": int(overlap)})
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    for k in ("th", "u", "v", "w", "p"):
        assert bits_equal(out[k], ref[k]), k
    # the first step after the copy-in pushes, the following ones are handed off
    assert all(p[1] == (1, case.ints["nsteps"] - 1) for p in parts), [p[1] for p in parts]


@pytest.mark.parametrize("name,px,py", [("dycore4", 2, 2), ("dycore4", 4, 2), ("dycore_full4", 3, 2)])
def test_peer_graph_replay_decomposed(name, px, py):
    """Decomposed steps replayed from CUDA graphs (hfb_run_graph) over the peer transport:
    the halo epochs live in device memory, so each replay of the captured push / signal /
    wait and epilogue hand-off sequence uses fresh epochs. Two replays of a 2-step graph
    equal the undecomposed oracle's 4 steps bit for bit; the exchanges are one push (the
    first step after the copy-in) and three epilogue hand-offs."""
    case, garr, out, parts = run_peer(name, px, py, per_step="graph")
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    for k in APPS[case.app].outputs:
        assert bits_equal(out[k], ref[k]), f"{name} {px}x{py}: {k} differs"
    assert all(p[1] == (1, 3) for p in parts), [p[1] for p in parts]


@pytest.mark.parametrize("px,py", [(2, 2), (3, 1)])
def test_peer_ordered_reduction_bit_exact(px, py):
    """Ordered reductions across processes: every rank gathers all tiles' column partials
    into global (j, i) order through peer memory and combines them in the acc-simulated
    order — the total is bit-identical to run_gpu_simulated's on every rank."""
    case, garr, _, parts = run_peer("reduction", px, py, ordered=True)
    accsim = run_oracle(case, {k: v.copy() for k, v in garr.items()})["total_accsim"]
    for p in parts:
        assert np.float64(p[3]).view(np.uint64) == np.float64(accsim).view(np.uint64)


def ckpt_worker(rank, world, port, px, py, phase, tmpdir, q):
    """phase 0: 2 steps then an HFBSTAT1 image per rank; phase 1: restore, 1 more step."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = PEER_CASES["dycore"]
        gnx, gny = global_extent(case)
        d = hfb.decomp_init(gnx, gny, case.ints["nz"], px, py, rank, halo=2)
        img = os.path.join(tmpdir, f"rank{rank}.hfbstate")
        if phase == 0:
            garr = make_inputs(case)
            eng = hfb.Engine("dycore", device=0)
            eng.set_decomposition(d)
            ints = dict(tile_ints(case, d), nsteps=2)
            for k, v in ints.items():
                eng.set(k, int(v))
            for k, v in case.reals.items():
                eng.set(k, float(v))
            for n, a in garr.items():
                eng.bind(n, np.ascontiguousarray(a[tile_slices(case.app, n, a, d)]))
            eng.attach_peers()
            eng.run("main")
            eng.save_state(img)
            q.put((rank, None, None))
        else:
            eng = hfb.Engine.from_state(img, device=0)
            eng.set("nsteps", 1)
            eng.set_decomposition(d)
            eng.attach_peers()
            eng.run("main")
            q.put((rank, {n: eng.array(n).copy() for n in ("th", "u", "v", "w", "p")}, None))
        dist.barrier()
        eng.close()
    except Exception as e:
        q.put((rank, None, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_peer_checkpoint_resume_per_rank(tmp_path):
    """Each rank writes its tile's MachineState image after 2 decomposed steps; fresh
    processes restore them, re-attach the peer transport and run 1 more step: the
    assembled tiles equal 3 undecomposed steps bit for bit."""
    px, py, world = 2, 2, 4
    ctx = mp.get_context("spawn")
    parts = None
    for phase in (0, 1):
        q = ctx.Queue()
        port = free_port()
        procs = [ctx.Process(target=ckpt_worker, args=(r, world, port, px, py, phase,
                                                       str(tmp_path), q)) for r in range(world)]
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
    case = PEER_CASES["dycore"]
    garr = make_inputs(case)
    ref = {k: v.copy() for k, v in garr.items()}
    ref_case = Case("ck", "dycore", dict(case.ints, nsteps=3), case.reals, case.fills)
    run_oracle(ref_case, ref)
    gnx, gny = global_extent(case)
    for rank, tiles, _ in parts:
        d = hfb.decomp_init(gnx, gny, case.ints["nz"], px, py, rank, halo=2)
        for k, t in tiles.items():
            want = ref[k][tile_slices(case.app, k, ref[k], d)]
            assert bits_equal(t.reshape(want.shape), want), (rank, k)


def c4_worker(rank, world, port, px, py, tmpdir, q):
    """One rank of the north-star grid split 4 x 2 (tiles 396 x 651 / 395 x 650): builds
    only its own tile of the synthetic state (global flat indices), runs `main_full`
    (copy-in, 2 full timesteps: one push, one epilogue hand-off, copy-out) and saves the
    tile's outputs for the parent."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1710_08616_b200 import synthetic
        gnx, gny, nz = C4
        d = hfb.decomp_init(gnx, gny, nz, px, py, rank, halo=2)
        eng = hfb.Engine("dycore", device=0)
        eng.set_decomposition(d)
        for k, v in dict(nx=int(d.nx), ny=int(d.ny), nz=nz, nsteps=2).items():
            eng.set(k, v)
        for k, v in dict(DYCORE_SCALARS, **PHYS_SCALARS).items():
            eng.set(k, float(v))
        box3 = [(0, nz), (d.i0, d.i0 + d.nx), (d.j0, d.j0 + d.ny)]
        tiles = {k: synthetic.field((nz, gnx, gny), *v, box=box3) for k, v in DYCORE_FILLS.items()}
        tiles.update({k: synthetic.field((gnx, gny), *v, box=box3[1:])
                      for k, v in PHYS_FILLS.items()})
        for n, a in tiles.items():
            eng.bind(n, a)
        eng.attach_peers()
        eng.run("main_full")
        for n, a in tiles.items():
            np.save(os.path.join(tmpdir, f"r{rank}_{n}.npy"), a)
        q.put((rank, eng.peer_stats(), (int(d.i0), int(d.j0), int(d.nx), int(d.ny)), None))
        dist.barrier()
        eng.close()
    except Exception as e:
        q.put((rank, None, None, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


C4 = (1581, 1301, 58)


def test_peer_c4_strong_scaling_tiles_4x2(tmp_path):
    """BASELINE configs[3] at 8 GPUs: the 1581 x 1301 x 58 grid as 4 x 2 tiles (396 x 651),
    one process per rank over the peer transport, two full timesteps (north_star step:
    dycore + HE-VI + column physics). The assembled tiles equal the undecomposed oracle
    bit for bit."""
    px, py = 4, 2
    world = px * py
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=c4_worker, args=(r, world, port, px, py, str(tmp_path), q))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        parts = [q.get(timeout=600) for _ in range(world)]
        for p in procs:
            p.join(timeout=120)
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
    errors = [e for *_, e in parts if e]
    assert not errors, errors
    assert sorted((r[2][2], r[2][3]) for r in parts)[-1] == (396, 651)
    assert all(p[1] == (1, 1) for p in parts), [p[1] for p in parts]
    case = Case("c4_full", "dycore_full", dict(nx=C4[0], ny=C4[1], nz=C4[2], nsteps=2),
                dict(DYCORE_SCALARS, **PHYS_SCALARS), dict(DYCORE_FILLS, **PHYS_FILLS))
    ref = make_inputs(case)
    run_oracle(case, ref)
    for rank, _, (i0, j0, nx, ny), _ in parts:
        for n in ("th", "u", "v", "w", "p", "colm"):
            t = np.load(tmp_path / f"r{rank}_{n}.npy")
            want = ref[n][..., i0:i0 + nx, j0:j0 + ny] if ref[n].ndim == 3 else \
                ref[n][i0:i0 + nx, j0:j0 + ny]
            assert bits_equal(t, want), f"rank {rank}: {n} differs"


@pytest.mark.parametrize("name,px,py,overlap", [("asuca", 2, 1, 1), ("asuca", 2, 2, 1),
                                                ("asuca", 3, 2, 1), ("asuca", 2, 2, 0),
                                                ("asuca_wide", 2, 2, 1)])
def test_peer_asuca_scheme_equals_single_domain(name, px, py, overlap):
    """The complete ASUCA step on a decomposed context (peer transport, one process per
    rank): each pass's stencil inputs are pushed into the neighbours' halo rings — the
    stage state for the tendencies, fu/fv and p/u/v for every first acoustic pass, pa for
    every second — on the communication stream while the pass runs over the columns 2
    cells inside the tile, then the boundary strips (overlap=0: exchange first, one
    full-span launch); the assembled tiles equal the undecomposed oracle bit for bit (the
    lateral damping band crosses tile edges)."""
    case, garr, out, parts = run_peer(name, px, py, options={"overlap": overlap})
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    for k in APPS[case.app].outputs:
        assert bits_equal(out[k], ref[k]), f"asuca {px}x{py}: {k} differs"
    # nsound = 6: per step 3 stage-state exchanges, 3 fu/fv, 11 p/u/v, 11 pa
    n = case.ints["nsteps"]
    assert all(p[1] == (28 * n, 0) for p in parts), [p[1] for p in parts]
    # per step 3 tendency passes, 22 acoustic passes (interior + 4 strips each when
    # overlapped) and 3 stage ends
    per_pass = 5 if overlap else 1
    assert all(p[5] == n * (25 * per_pass + 3) for p in parts), [p[5] for p in parts]


def test_peer_asuca_graph_replay():
    """asuca_step replayed from a CUDA graph on the decomposed context (device-side halo
    epochs): equal to the undecomposed oracle."""
    case, garr, out, parts = run_peer("asuca", 2, 2, per_step="graph")
    ref = {k: v.copy() for k, v in garr.items()}
    run_oracle(case, ref)
    for k in APPS[case.app].outputs:
        assert bits_equal(out[k], ref[k]), k


def test_bench_multi_rank_path_on_one_gpu():
    """bench.py's multi-rank path (torchrun, 2 ranks, peer transport, graph-replayed timed
    region, e2e) with both ranks on this one GPU (--one-gpu-test): it must finish and print
    one JSON line — every rank runs the same number of steps (the warm-up count is agreed
    over the ranks), or the pairwise exchanges deadlock."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items() if not k.startswith("HFB_")}
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(free_port()), str(root / "bench.py"), "--gpus", "2", "--steps", "4",
                        "--warmup", "3", "--tile512", "--one-gpu-test", "--no-secondary"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["halo"]["bytes_per_step_rank0"] > 0
