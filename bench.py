#!/usr/bin/env python3
"""Benchmark: one full ASUCA-style timestep per step — the fused dynamical core
(flux-limited advection, pressure gradient + divergence, HE-VI vertically implicit Thomas
solve) plus the column physics (`full_step`, apps/dycore/dycore.h90).

Workload (north_star; BASELINE configs[3] at N=1, configs[4] per GPU for N > 1): a
1581 x 1301 x 58 grid per GPU, fp64, synthetic state (SURVEY §8(d) SplitMix64 fields).
Metric: grid-point updates per second per timestep (nx*ny*nz / t_step, whole job) and the
HBM-roofline fraction of the dominant kernel.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--strong | --tile512] [--entry full_step|dycore_step]
                  [--transport peer|nccl]

N > 1 runs under torchrun, one rank per GPU: a 2-D (px x py) horizontal block
decomposition, WEAK scaling (a 1581 x 1301 x 58 tile per GPU, configs[4]); `--strong`
splits the one 1581 x 1301 x 58 grid (configs[3]). The halo exchange uses the peer-memory
transport (push kernels storing into the neighbours' halo rings over NVLink/NVSwitch,
CUDA IPC-mapped buffers, release/acquire flags); `--transport nccl` selects NCCL
send/recv instead.
`--impl reference` times the reference's own CPU path (oracle/_ref/hft_ref: the
reference interpreter built from /root/reference/proj/src) on the host cores.
The bench reads no HFB_* environment variable and refuses to run if one is set: every
switch is a command-line flag, so a result cannot depend on a hidden knob.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

NX, NY, NZ = 1581, 1301, 58  # the production domain (north_star; BASELINE configs[3]/[4])
C2_NX, C2_NY = 512, 512     # BASELINE configs[1] (--tile512)
METRIC = "grid-point updates/sec per timestep"
UNIT = "grid-point updates/s"
GRIDS = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}
# compulsory HBM bytes per grid point and step of each native kernel:
# the fused step reads rho,th,u,v,w,p and writes th',u',v',w',p' (11 x 8 B); the full
# step adds, per COLUMN, tsfc and colm read and colm written (3 x 8 B); the split
# variant's advect reads th,u,v,w / writes th' (5 x 8 B) and acoustic reads
# rho,th,u,v,w,p / writes u',v',w',p' (10 x 8 B)
BYTES_PER_POINT = {"dycore_step": 88, "full_step": 88, "dycore_advect": 40,
                   "dycore_acoustic": 80, "hfk0_diffuse_step": 24}
BYTES_PER_COLUMN = {"full_step": 24}
# asuca_step (apps/dycore/asuca.h90, nsound = 6): per RK3 stage the slow tendencies read
# rho, th, u, v, w and write 5 tendencies (80 B); every short step's RK2 pass A reads
# u, v, w, p, rho, th, fu, fv, fw and writes pa (80 B), pass B also reads pa and writes
# u, v, w, p (112 B); the stage end reads thb, fth, rhob, frho and writes th, rho (48 B):
# 3 x (80 + 48) + (2 + 3 + 6) x (80 + 112) = 2496 B per point and step
ASUCA_KERNEL_BYTES = {"asuca_tend": 80, "asuca_acoustic_a": 80, "asuca_acoustic_b": 112,
                      "asuca_stage_end": 48}
ASUCA_BYTES_PER_POINT = 3 * (80 + 48) + 11 * (80 + 112)


def alg_bytes(kernel, nx, ny, nz):
    """algorithmic (compulsory) HBM bytes of one launch over an nx x ny x nz tile"""
    return BYTES_PER_POINT[kernel] * nx * ny * nz + BYTES_PER_COLUMN.get(kernel, 0) * nx * ny
L2_BYTES = 126 * 2**20


def cpu_model():
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device, interval_ms=20):
        self.device = device
        self.interval_ms = interval_ms
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi may take a while to start: wait for its first sample so the
            # timed region is bracketed by samples
            deadline = time.perf_counter() + 10.0
            while not self.rows and time.perf_counter() < deadline and self.proc.poll() is None:
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None
        self.t0 = self.t1 = time.perf_counter()
        return self

    def start(self):  # the timed region begins (after the ranks' barrier)
        self.t0 = time.perf_counter()

    def stop(self):  # the timed region ended (after the device synchronize)
        self.t1 = time.perf_counter()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append((time.perf_counter(), parts))

    def __exit__(self, *a):
        if self.proc:
            # at least one sample after the region ended
            deadline = self.t1 + 2.0
            while (not self.rows or self.rows[-1][0] <= self.t1) and \
                    time.perf_counter() < deadline and self.proc.poll() is None:
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def window(self):
        """Samples inside the timed region plus the nearest one on each side (the region
        can be shorter than the sampling interval)."""
        inside = [r for t, r in self.rows if self.t0 <= t <= self.t1]
        before = [r for t, r in self.rows if t < self.t0][-1:]
        after = [r for t, r in self.rows if t > self.t1][:1]
        return before + inside + after

    def summary(self):
        rows = self.window()
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[q] for r in rows for q in range(4)
                          if r[2 + q].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows),
                "window_ms": round((self.t1 - self.t0) * 1e3, 2)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def decompose(eng, d, n, transport, dist):
    """Attach the rank's tile; NCCL needs the shared unique id now, the peer transport
    maps the neighbours' buffers once the state is bound (Engine.attach_peers)."""
    if n == 1:
        return
    if transport == "nccl":
        import paper_1710_08616_b200 as hfb
        obj = [hfb.runtime.nccl_unique_id() if d.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng.set_decomposition(d, obj[0])
    else:
        eng.set_decomposition(d)


def make_state(eng, d, gnx, gny, physics, asuca=False):
    """Bind the synthetic state of this rank's tile (global-flat-indexed fields, pinned
    host buffers); `physics` adds the column-physics fields of the full timestep, `asuca`
    the ASUCA scheme's scalars (set before the peers are attached: the export then maps
    the scheme's exchanged scratch)."""
    from paper_1710_08616_b200 import synthetic
    box = [(0, NZ), (d.i0, d.i0 + d.nx), (d.j0, d.j0 + d.ny)]
    arrs = {k: synthetic.field((NZ, gnx, gny), *v, box=box, order="F")
            for k, v in synthetic.DYCORE_FILLS.items()}
    scalars = dict(synthetic.DYCORE_SCALARS)
    if physics:
        box2 = box[1:]
        arrs.update({k: synthetic.field((gnx, gny), *v, box=box2, order="F")
                     for k, v in synthetic.PHYS_FILLS.items()})
        scalars.update(synthetic.PHYS_SCALARS)
    if asuca:
        scalars.update(synthetic.asuca_params(NZ))
    for k, v in dict(nx=int(d.nx), ny=int(d.ny), nz=NZ, nsteps=1).items():
        eng.set(k, v)
    for k, v in scalars.items():
        eng.set(k, v)
    for k, a in arrs.items():
        eng.bind(k, a, pin=True)
    return arrs


def secondary(local, steps=20, warmup=5):
    """Single-GPU, device-resident timings of the other BASELINE configs (reported beside
    the headline; same CUDA-event method over `steps` back-to-back steps replayed from one
    CUDA graph)."""
    import torch
    import paper_1710_08616_b200 as hfb
    from paper_1710_08616_b200 import synthetic
    hbm, _ = peaks()
    out = {}
    runs = [("C1 dycore step 128x128x58 (BASELINE configs[0])", "dycore", "dycore_step", 128, 128),
            ("C2 dycore step 512x512x58 (BASELINE configs[1])", "dycore", "dycore_step", 512, 512),
            ("C2 dycore with Wicker-Skamarock RK3 (3 stages) 512x512x58", "dycore", "rk3_step",
             512, 512),
            ("C3 full timestep + column physics 1024x1024x58 (BASELINE configs[2])", "dycore",
             "full_step", 1024, 1024),
            ("C4 dycore step without physics 1581x1301x58", "dycore", "dycore_step", 1581, 1301),
            ("reference kernel: diffusion step 1581x1301x58", "diffusion", "diffuse_step",
             1581, 1301),
            ("ASUCA time scheme (RK3 + 11 RK2 HE-VI acoustic short steps + damping + limited "
             "advection of rho, theta, u, v, w) 1581x1301x58", "dycore", "asuca_step", 1581, 1301)]
    for label, prog, entry, nx, ny in runs:
        eng = hfb.Engine(prog, device=local)
        shape = (NZ, nx, ny)
        for k, v in dict(nx=nx, ny=ny, nz=NZ, nsteps=1).items():
            eng.set(k, v)
        if prog == "dycore":
            for k, v in dict(synthetic.DYCORE_SCALARS, **synthetic.PHYS_SCALARS).items():
                eng.set(k, v)
            arrs = {k: synthetic.field(shape, *v, order="F")
                    for k, v in synthetic.DYCORE_FILLS.items()}
            if entry == "full_step":
                arrs.update({k: synthetic.field((nx, ny), *v, order="F")
                             for k, v in synthetic.PHYS_FILLS.items()})
            if entry == "asuca_step":
                for k, v in synthetic.asuca_params(NZ).items():
                    eng.set(k, v)
            # RK3: stage 1 as the single step (88 B/pt); stages 2-3 also read the base
            # th, u, v, w, p (128 B/pt each)
            abytes = (88 + 2 * 128) * nx * ny * NZ if entry == "rk3_step" else \
                ASUCA_BYTES_PER_POINT * nx * ny * NZ if entry == "asuca_step" else \
                alg_bytes(entry, nx, ny, NZ)
        else:
            eng.set("coef", 0.1)
            arrs = {"t_old": synthetic.field(shape, 1, 280.0, 10.0, order="F"),
                    "t_new": np.zeros(shape, order="F")}
            abytes = alg_bytes("hfk0_diffuse_step", nx, ny, NZ)
        for k, a in arrs.items():
            eng.bind(k, a)
            eng.copy_to_device(k)
        stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", local))
        nst = 5 if entry == "asuca_step" else steps  # ~0.1 s per asuca step at C4
        for _ in range(min(warmup, nst)):
            eng.enqueue(entry)
        eng.synchronize()
        # the timed steps replay one CUDA graph (as the headline): captured for both buffer
        # sides first
        eng.enqueue_graph(entry, nst)
        eng.enqueue_graph(entry, nst)
        eng.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.enqueue_graph(entry, nst)
        e1.record(stream)
        eng.synchronize()
        ms = e0.elapsed_time(e1) / nst
        kern = None
        if entry == "asuca_step":  # per-kernel device times of one more step
            eng.profile(True, clear=True)
            eng.profile(True)
            eng.enqueue(entry)
            eng.synchronize()
            eng.profile(False)
            kern = {}
            for kname, b in ASUCA_KERNEL_BYTES.items():
                t, nl = eng.kernel_time(kname)
                if nl:
                    kern[kname] = {"launches_per_step": nl, "ms_each": round(t / nl, 4),
                                   "alg_bytes_per_point": b,
                                   "GBps": round(b * nx * ny * NZ / (t / nl / 1e3) / 1e9, 1)}
        pts = nx * ny * NZ
        gbs = abytes / (ms / 1e3) / 1e9
        out[label] = {"entry": entry, "ms_per_step": round(ms, 4),
                      "value": round(pts / (ms / 1e3), 1), "unit": UNIT,
                      "alg_bytes_per_step": abytes, "achieved_GBps": round(gbs, 1),
                      "frac_of_measured_hbm": round(gbs / hbm, 4),
                      "frac_of_nominal_8TBps": round(gbs / 8000.0, 4), "steps": nst,
                      "timed_steps": f"{nst} steps replayed from one CUDA graph"}
        if kern:
            out[label]["kernels"] = kern
        eng.close()
        del arrs
    return out


def cpu_baseline_port(seconds_budget=20.0, asuca=False):
    """The C restatement (oracle/, KIJ storage, OpenMP over j on every host core) timed on
    a bounded sample of the same workload: whole full timesteps of a 512x512x58 block
    (the per-point cost does not depend on the block size; the C4 grid would need ~20 GB
    of host memory for the oracle's state and scratch); ASUCA steps of a 128x128x58 block
    for --entry asuca_step."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle
    from paper_1710_08616_b200 import synthetic
    cores = os.cpu_count() or 1
    oracle.set_threads(cores)
    sx, sy = (128, 128) if asuca else (C2_NX, C2_NY)
    a = {k: synthetic.field((NZ, sx, sy), *v, order="F") for k, v in synthetic.DYCORE_FILLS.items()}
    a.update({k: synthetic.field((sx, sy), *v, order="F") for k, v in synthetic.PHYS_FILLS.items()})
    prm = dict(synthetic.DYCORE_SCALARS, **synthetic.PHYS_SCALARS)
    ap = synthetic.asuca_params(NZ)
    prm.update({k: v for k, v in ap.items() if isinstance(v, float)})
    ints = {k: v for k, v in ap.items() if isinstance(v, int)}

    def one():
        if asuca:
            oracle.asuca_run(1, prm, ints, a["rho"], a["th"], a["u"], a["v"], a["w"], a["p"])
            return
        oracle.full_run(1, prm, a["rho"], a["th"], a["u"], a["v"], a["w"], a["p"], a["tsfc"],
                        a["colm"])
    one()  # warm (scratch allocation, page faults)
    steps, t0 = 0, time.perf_counter()
    while True:
        one()
        steps += 1
        el = time.perf_counter() - t0
        if el > seconds_budget / 2 or steps >= 20:
            break
    return {"value": sx * sy * NZ * steps / el, "unit": UNIT, "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"{steps} {'ASUCA steps (asuca_step)' if asuca else 'full timesteps (full_step)'}"
                      f" of a {sx}x{sy}x{NZ} block "
                      f"(oracle/hfb_oracle.c, KIJ order, OpenMP {cores} threads), {el:.2f} s"}


def bench_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1710_08616_b200 as hfb

    rank, world, local = dist_env()
    n = args.gpus

    def trace(what):  # --trace: phase markers on stderr (debugging multi-rank runs)
        if args.trace:
            print(f"[bench rank {rank}] {what} t={time.perf_counter():.2f}", file=sys.stderr,
                  flush=True)
    if world != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world}")
    if n not in GRIDS:
        raise SystemExit("--gpus must be 1, 2, 4 or 8")
    px, py = GRIDS[n]
    entry = args.entry
    physics = entry == "full_step"
    asuca = entry == "asuca_step"
    # --one-gpu-test (testing only): every rank on cuda:0, gloo for the host-side
    # collectives — exercises the multi-rank path (peer transport) on a one-GPU box
    one_gpu = args.one_gpu_test
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if n > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    trace("process group up")
    eng = hfb.Engine("dycore", device=local)
    # weak scaling (default): a 1581 x 1301 tile per GPU; --strong: the C4 grid split
    tnx, tny = (C2_NX, C2_NY) if args.tile512 else (NX, NY)  # weak-scaling tile
    gnx, gny = (NX, NY) if args.strong else (tnx * px, tny * py)
    d = hfb.decomp_init(gnx, gny, NZ, px, py, rank, halo=2)
    decompose(eng, d, n, args.transport, dist)
    arrs = make_state(eng, d, gnx, gny, physics, asuca)
    transport_note = None
    if n > 1 and args.transport == "peer":
        # the peer transport maps the neighbours' buffers by CUDA IPC; if that fails on any
        # rank (e.g. no peer access between the devices), every rank falls back to NCCL
        err = ""
        try:
            eng.attach_peers()
        except Exception as e:  # noqa: BLE001 - reported in the JSON line
            err = repr(e)[:200]
        t = torch.tensor([0.0 if err else 1.0], device="cpu" if one_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if t.item() < 1.0:
            if one_gpu:
                raise SystemExit(f"peer attach failed on one GPU: {err}")
            eng.close()
            args.transport = "nccl"
            transport_note = f"peer transport unavailable ({err or 'on another rank'}): NCCL"
            eng = hfb.Engine("dycore", device=local)
            decompose(eng, d, n, "nccl", dist)
            arrs = make_state(eng, d, gnx, gny, physics, asuca)
    trace("state bound, peers attached")
    for k in arrs:
        eng.copy_to_device(k)
    eng.synchronize()

    stream = torch.cuda.ExternalStream(eng.stream, device=torch.device("cuda", local))

    def barrier():
        if n > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up: W steps, extended to >= 0.4 s of back-to-back steps so the timed
    # region sees the SUSTAINED (power-capped) clock state, not the burst one; the timed
    # K steps replay ONE CUDA graph (hfb_enqueue_graph: the native host driver's steps,
    # halo exchange included for N > 1), captured here for both buffer sides ------------
    # (NCCL send/recv is not graph-captured: that transport keeps the launch loop)
    use_graph = n == 1 or args.transport == "peer"

    def run_steps():
        if use_graph:
            return eng.enqueue_graph(entry, args.steps).native_launches
        return sum(eng.enqueue(entry).native_launches for _ in range(args.steps))

    for _ in range(args.warmup):
        eng.enqueue(entry)
    eng.synchronize()
    trace("warm-up steps done")
    run_steps()  # graph capture (+ K steps)
    run_steps()  # the other buffer side when K is odd
    eng.synchronize()
    trace("graphs captured")
    w0 = time.perf_counter()
    for _ in range(args.warmup):
        eng.enqueue(entry)
    eng.synchronize()
    per = (time.perf_counter() - w0) / max(1, args.warmup)
    if n > 1:  # every rank must run the same number of steps (the exchanges pair up)
        t = torch.tensor([per], device="cpu" if one_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        per = float(t.item())
    extra = max(0, int(0.4 / max(per, 1e-6)) - args.warmup)
    trace(f"per-step {per * 1e3:.3f} ms, {extra} more warm-up steps")
    for _ in range(extra):
        eng.enqueue(entry)
    warmup_run = 2 * args.warmup + extra + 2 * args.steps
    eng.synchronize()
    trace("sustained warm-up done")

    # ---- device-resident timed region: K timesteps ------------------------------------
    t_ev0 = torch.cuda.Event(enable_timing=True)
    t_ev1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(local, args.smi_ms) as clocks:  # nvidia-smi running before the region
        barrier()
        trace("timed region starts")
        clocks.start()
        t_ev0.record(stream)
        launches += run_steps()
        t_ev1.record(stream)
        eng.synchronize()
        clocks.stop()
    barrier()
    ms = t_ev0.elapsed_time(t_ev1)
    trace("timed region done")
    # per-kernel device times from a second pass of the same K steps with CUDA events
    # around every launch (hfb_profile); kept out of the timed region, whose events
    # would otherwise add ~2% to the step
    eng.profile(True, clear=True)
    eng.profile(True)
    barrier()
    for _ in range(args.steps):
        eng.enqueue(entry)
    eng.synchronize()
    barrier()
    eng.profile(False)
    kernel_bytes = ASUCA_KERNEL_BYTES if asuca else BYTES_PER_POINT
    kt = {k: eng.kernel_time(k) for k in kernel_bytes}
    kt = {k: v for k, v in kt.items() if v[1] > 0}
    # the tolerance mode side by side (hfb_set_option "arith" "fma": the same fused step
    # with FMA contraction, within 1e-12 per field of the reference after one step,
    # tests/test_gpu_tolerance.py): the same K steps, graph-replayed, timed right after K
    # more steps of the exact build, so both see the same (later, hotter) clock state
    def timed_region():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        run_steps()
        e1.record(stream)
        eng.synchronize()
        barrier()
        return e0.elapsed_time(e1)
    if asuca:  # the tolerance build exists for the fused dycore step only
        ms_exact2 = ms_fma = ms
    else:
        ms_exact2 = timed_region()
        eng.set_option("arith", "fma")
        run_steps()
        run_steps()
        ms_fma = timed_region()
        eng.set_option("arith", "exact")
    trace("tolerance-mode region done")
    ms_local = ms
    if n > 1:
        t = torch.tensor([ms], device="cpu" if one_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if n > 1:
        t = torch.tensor([ms_fma, ms_exact2], device="cpu" if one_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_fma, ms_exact2 = float(t[0].item()), float(t[1].item())
    pts_step = gnx * gny * NZ
    value = pts_step * args.steps / (ms / 1e3)

    # ---- roofline of the dominant kernel (live CUDA events over the timed region) -------
    hbm, src = peaks()
    dom = max(kt, key=lambda k: kt[k][0])
    dom_ms, dom_n = kt[dom]
    tnx_l, tny_l = int(d.nx), int(d.ny)
    # one step of the tile is one launch (N=1) or the interior launch plus four boundary
    # strips (decomposed, halo exchange overlapped): the kernel's device time per STEP
    # moves the tile's algorithmic bytes
    abytes = (ASUCA_KERNEL_BYTES[dom] * tnx_l * tny_l * NZ if asuca
              else alg_bytes(dom, tnx_l, tny_l, NZ))
    per_step_prof = dom_ms / args.steps
    if asuca:  # several launches of the dominant pass per step: its time per LAUNCH
        per_step = dom_ms / dom_n
        timing = "per-launch events (profiled pass), per launch"
    elif dom_n == args.steps:  # the step is this one launch: the timed region's CUDA events
        per_step = ms_local / args.steps  # (launch stream) / launches — conservative, it
        timing = "timed-region events / launches"  # includes the gaps between launches
    else:
        per_step = per_step_prof
        timing = "per-launch events (profiled pass)"
    achieved = abytes / (per_step / 1e3) / 1e9
    # measured DRAM traffic of this kernel on THIS tile shape (ncu --set full capture,
    # profiles/traffic.json keyed by "<kernel> <nx>x<ny>x<nz>"); null when not captured
    traffic = None
    tkey = f"{dom} {tnx_l}x{tny_l}x{NZ}"
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        rec = json.loads(tp.read_text()).get(tkey)
        traffic = rec["dram_bytes"] if isinstance(rec, dict) else None
    ach_fma = abytes / (ms_fma / args.steps / 1e3) / 1e9
    tolerance_mode = {"arith": "fma", "ms_per_step": round(ms_fma / args.steps, 5),
                      "exact_ms_per_step_same_state": round(ms_exact2 / args.steps, 5),
                      "value": round(pts_step * args.steps / (ms_fma / 1e3), 1), "unit": UNIT,
                      "roofline_frac": round(ach_fma / hbm, 4),
                      "achieved_GBps": round(ach_fma, 1),
                      "tolerance": "<= 1e-12 relative (normwise) per field after one step; "
                                   "<= 1e-10 after 100 steps (tests/test_gpu_tolerance.py)",
                      "note": "opt-in (hfb_set_option arith=fma); the headline is the "
                              "default, bit-exact build"}
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic, "traffic_key": tkey,
                "kernel": dom, "frac_of_nominal_8TBps": round(achieved / 8000.0, 4),
                "peak_source": src, "algorithmic_bytes_per_launch": abytes,
                "algorithmic_bytes": f"{kernel_bytes[dom]} B/point x {tnx_l}x{tny_l}x{NZ}"
                                     + (f" + {BYTES_PER_COLUMN[dom]} B/column x {tnx_l}x{tny_l}"
                                        if dom in BYTES_PER_COLUMN else "")
                                     + (" per launch" if asuca else ""),
                "launches_per_step": dom_n // args.steps,
                "algorithmic_bytes_per_step": (ASUCA_BYTES_PER_POINT * tnx_l * tny_l * NZ
                                               if asuca else abytes),
                "step_frac": round(ASUCA_BYTES_PER_POINT * tnx_l * tny_l * NZ /
                                   (ms_local / args.steps / 1e3) / 1e9 / hbm, 4)
                if asuca else None,
                "kernel_ms_avg": round(per_step, 5), "timing": timing,
                "kernel_ms_profiled": round(per_step_prof, 5),
                "share_of_step": round(min(1.0, per_step_prof / (ms_local / args.steps)), 3),
                "kernels": {k: {"ms_avg": round(v[0] / args.steps, 5),
                                "launches_per_step": v[1] // args.steps,
                                "GBps": round(kernel_bytes[k] * tnx_l * tny_l * NZ * v[1] /
                                              args.steps / (v[0] / args.steps / 1e3) / 1e9, 1)
                                if asuca else
                                round(alg_bytes(k, tnx_l, tny_l, NZ) /
                                      (v[0] / args.steps / 1e3) / 1e9, 1)}
                            for k, v in kt.items()}}

    # ---- end to end through the public API with host buffers --------------------------
    # one e2e step = one call of the program's main entry (transferHere copy-in of the
    # state arrays from pinned host memory, `nsteps` timesteps, copy-out), as the
    # generated host code does (codegen.cpp:570-600)
    main_entry = "main_full" if physics else "main_asuca" if asuca else "main"
    e2e_nsteps = 10 if asuca else 100
    eng2 = hfb.Engine("dycore", device=local)
    decompose(eng2, d, n, args.transport, dist)
    arrs2 = make_state(eng2, d, gnx, gny, physics, asuca)
    if n > 1 and args.transport == "peer":
        eng2.attach_peers()
    eng2.set("nsteps", e2e_nsteps)
    trace("e2e engine ready")
    eng2.run(main_entry)  # warm-up call
    trace("e2e warm-up call done")
    arrs2 = make_state(eng2, d, gnx, gny, physics, asuca)
    eng2.set("nsteps", e2e_nsteps)
    e2e_calls = max(1, min(3, args.steps // 10))
    xb0 = eng2.transfer_bytes()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_calls):
        eng2.run(main_entry)
    t1 = time.perf_counter()
    xb1 = eng2.transfer_bytes()
    e2e_s = t1 - t0
    if n > 1:
        t = torch.tensor([e2e_s], device="cpu" if one_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # bytes the runtime actually moved per call (rank 0's tile): every state field in; out,
    # the ones the steps rewrote (rho and tsfc are untouched on the device, so their
    # copy-out is a no-op: host and device already hold the same bytes)
    h2d = (xb1[0] - xb0[0]) // e2e_calls
    d2h = (xb1[1] - xb0[1]) // e2e_calls
    e2e = {"value": pts_step * e2e_nsteps * e2e_calls / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "step": f"one `{main_entry}` call through the C ABI: copy-in of the {len(arrs2)} "
                   f"pinned host fields, {e2e_nsteps} timesteps, copy-out",
           "timesteps_per_step": e2e_nsteps, "calls": e2e_calls}
    halo = eng.halo_bytes()
    eng2.close()
    eng.close()

    if rank == 0:
        what = ("full timestep (dycore + HE-VI + column physics)" if physics
                else "ASUCA time scheme (RK3 + 11 RK2 HE-VI acoustic short steps + damping + "
                     "limited advection of rho, theta, u, v, w; 2496 B/pt)" if asuca
                else "dycore step (advection + HE-VI)")
        if args.strong:
            wl = f"{what} {NX}x{NY}x{NZ} split over {n} GPU(s) (BASELINE configs[3], strong)"
        elif args.tile512:
            wl = f"{what} {tnx}x{tny}x{NZ} per GPU (BASELINE configs[1] grid)"
        elif n == 1:
            wl = f"{what} {NX}x{NY}x{NZ} on 1 GPU (north_star; BASELINE configs[3] at N=1)"
        else:
            wl = f"{what} {tnx}x{tny}x{NZ} per GPU (BASELINE configs[4], weak)"
        out = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": n,
               "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": round(ms / args.steps, 5), "higher_is_better": True,
               "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
               "dtype": "f64",
               "data": "synthetic (SplitMix64 fields, SURVEY §8(d))",
               "config": {"workload": wl, "entry": entry,
                          "global_grid": [gnx, gny, NZ], "decomposition": f"{px}x{py}",
                          "transport": args.transport if n > 1 else None,
                          "transport_note": transport_note,
                          "warmup_steps_run": warmup_run,
                          "timed_steps": f"{args.steps} steps replayed from one CUDA graph"
                          if use_graph else f"{args.steps} enqueued steps",
                          "timed_region_ms": round(ms, 3),
                          "column_sums": "thread per column, the K sum in the dialect's "
                                         "left-to-right order inside the fused step (bit-exact; "
                                         "no warp-level tree reduction)" if physics else None,
                          "l2": f"inputs larger than L2: "
                                f"{6 * tnx_l * tny_l * NZ * 8 / 2**30:.2f} GiB state + "
                                f"{5 * tnx_l * tny_l * NZ * 8 / 2**30:.2f} GiB outputs per "
                                f"step and GPU vs 126 MB L2 (no flush needed)"},
               "roofline": roofline, "tolerance_mode": None if asuca else tolerance_mode,
               "e2e": e2e,
               "gpu_launches": launches,
               "clocks": clocks.summary(), "halo_bytes": halo}
        if n > 1:  # rank 0's halo traffic (sent + received) per step and its rate
            hps = halo / (warmup_run + 2 * args.steps)
            out["halo"] = {"bytes_per_step_rank0": int(hps),
                           "GBps_rank0": round(hps / (ms / args.steps / 1e3) / 1e9, 2)}
        out["cpu_baseline"] = cpu_baseline_port(asuca=asuca) if n == 1 else None
        if n == 1 and not args.no_secondary:
            out["other_configs"] = secondary(local)
        print(json.dumps(out), flush=True)
    if n > 1:
        dist.destroy_process_group()


def bench_reference(args):
    """The reference's own CPU path: its binary64 interpreter (oracle/_ref/hft_ref, compiled
    from /root/reference/proj/src) running this repo's dycore app (apps/dycore, the
    reference dialect) through run_reference, entry main_full with nsteps = 1 (the full
    timestep). It is single-threaded by design, so every host core runs one
    independent interpreter over its own SAMPLE_NX x SAMPLE_NY x 58 column block of the
    workload. A step's time is the slowest interpreter's own run_reference time
    (the harness times the call; process start-up and .h90 parsing are excluded)."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    hft = ROOT / "oracle" / "_ref" / "hft_ref"
    if not hft.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "ref"], check=True)
    from paper_1710_08616_b200 import synthetic
    cores = os.cpu_count() or 1
    physics = args.entry == "full_step"
    asuca = args.entry == "asuca_step"
    sx, sy = (8, 8) if asuca else (16, 16)  # an ASUCA step is ~30x a full step's work
    tmp = Path(tempfile.mkdtemp(prefix="hftref_"))
    scen = tmp / "dycore.sc"
    lines = [f"source {ROOT / 'apps/dycore/dyn_state.h90'}",
             f"source {ROOT / 'apps/dycore/dycore.h90'}"]
    if asuca:
        lines.append(f"source {ROOT / 'apps/dycore/asuca.h90'}")
    lines += ["mode ref",
              f"entry {'main_full' if physics else 'main_asuca' if asuca else 'main'}",
              "max_steps 2000000000", f"int dyn_state nx {sx}", f"int dyn_state ny {sy}",
              f"int dyn_state nz {NZ}", "int dyn_state nsteps 1"]
    scal = dict(synthetic.DYCORE_SCALARS, **(synthetic.PHYS_SCALARS if physics else {}))
    if asuca:
        ap = synthetic.asuca_params(NZ)
        lines += [f"int dyn_state {k} {v}" for k, v in ap.items() if isinstance(v, int)]
        scal.update({k: v for k, v in ap.items() if isinstance(v, float)})
    fills = dict(synthetic.DYCORE_FILLS, **(synthetic.PHYS_FILLS if physics else {}))
    lines += [f"real dyn_state {k} {float(v).hex()}" for k, v in scal.items()]
    lines += [f"fill dyn_state {k} {s} {float(o).hex()} {float(c).hex()}"
              for k, (s, o, c) in fills.items()]
    scen.write_text("\n".join(lines) + "\n")

    def one_step():
        procs = [subprocess.Popen([str(hft), str(scen)], stdout=subprocess.PIPE, text=True)
                 for _ in range(cores)]
        secs = []
        for p in procs:
            out, _ = p.communicate()
            if p.returncode != 0:
                raise RuntimeError("reference interpreter failed")
            rec = [json.loads(ln) for ln in out.splitlines() if ln.startswith('{"seconds"')]
            secs.append(rec[-1]["seconds"])
        return max(secs)  # the interpreters run concurrently: the slowest one's run time

    for _ in range(args.warmup):
        one_step()
    el = sum(one_step() for _ in range(args.steps))
    value = cores * sx * sy * NZ * args.steps / el
    sample = (f"{cores} concurrent reference interpreters (run_reference, 1 thread each), "
              f"each one {'full timestep (main_full)' if physics else 'ASUCA step (main_asuca)' if asuca else 'dycore step'} of its "
              f"own {sx}x{sy}x{NZ} block of the {NX}x{NY}x{NZ} workload; time = the slowest "
              f"interpreter's run_reference call (process start and .h90 parsing excluded)")
    out = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (SplitMix64 fields, SURVEY §8(d))", "impl": "reference",
           "config": {"workload": f"{'full timestep' if physics else 'ASUCA step' if asuca else 'dycore step'} "
                                  f"{NX}x{NY}x{NZ} (north_star), sampled as {cores} blocks of "
                                  f"{sx}x{sy}x{NZ}", "entry": args.entry,
                      "sample": f"{cores} x {sx}x{sy}x{NZ} blocks"},
           "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": cores,
                            "kind": "reference", "sample": sample},
           "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    bad = sorted(k for k in os.environ if k.startswith("HFB_"))
    if bad:
        raise SystemExit(f"bench.py refuses to run with HFB_* environment variables set "
                         f"({', '.join(bad)}): every switch is a command-line flag")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--entry", default="full_step",
                    choices=["full_step", "dycore_step", "asuca_step"],
                    help="the timestep: full (dycore + column physics, default), dycore only, "
                         "or the ASUCA time scheme (use --steps 10: ~0.07 s per step at C4)")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling of the 1581x1301x58 grid (default: weak, a "
                         "1581x1301x58 tile per GPU)")
    ap.add_argument("--tile512", action="store_true",
                    help="a 512x512x58 tile per GPU (BASELINE configs[1] grid)")
    ap.add_argument("--c4-tiles", action="store_true", help=argparse.SUPPRESS)  # the default
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="halo exchange for N > 1 (peer: P2P stores + flags; nccl: send/recv)")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the single-GPU timings of the other BASELINE configs")
    ap.add_argument("--one-gpu-test", action="store_true",
                    help="testing only: every rank on cuda:0 (multi-rank path on one GPU)")
    ap.add_argument("--smi-ms", type=int, default=20, help="nvidia-smi sampling interval")
    ap.add_argument("--trace", action="store_true", help="phase markers on stderr")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
