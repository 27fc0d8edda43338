#!/usr/bin/env python
"""Benchmark of the hot path: one step = one complete solve (§4 cycle
from the initial state to termination) of the bench workload, inputs resident
in HBM.  Prints ONE JSON line (rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C3|C2|C3s]
    python bench.py --impl reference ...     # the CPU oracle on a bounded sample

Metric (BASELINE.json): active edge-updates/s = sum over cycles of (live active
edges + live phantom edges) / solve time; also reported: solve
time, and achieved HBM GB/s of the cycle kernel against MEASURED_PEAKS.json.
Multi-GPU (N > 1): `--gpus N` without torchrun re-launches this script under
torch.distributed.run with N ranks (one per GPU); under torchrun WORLD_SIZE
must equal N.  Default partition: the ONE instance cut into N z-slabs (SURVEY
§8(e); boundary fused over NVLink peer memory in one persistent kernel per GPU,
`--halo copy` for NCCL send/recv per cycle) — strong scaling; `--partition
replicas` solves an independent seed per rank instead (weak scaling).  The time
is the max over ranks of the device time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "active edge-updates/s and solve time on Z^d cubes; achieved HBM GB/s"
UNIT = "edge-updates/s"
WORKLOADS = {
    "C3": {"shape": (256, 256, 256), "desc": "configs[2]: 3D 256^3 cube, f1,f2 ~ U{1..10}, A = face x=0, "
                                             "B = face x=255, M = M_bind, 1 GPU"},
    "C2": {"shape": (1024, 1024), "desc": "configs[1]: 2D 1024^2, f1,f2 ~ U{1..10}, A = left face, B = right face, "
                                          "M = M_bind"},
    "C3s": {"shape": (128, 128, 128), "desc": "128^3 cube (reduced C3 for quick runs), M = M_bind"},
    "C5": {"shape": (1024, 1024, 1024), "desc": "configs[4]: 3D 1024^3 cube, f1,f2 ~ U{1..10}, face x=0 -> face "
                                                "x=1023, M = M_bind; unsliced on one B200 (about 105 GB of HBM) or "
                                                "z-slabs over N GPUs with --partition slabs"},
    "C5z8": {"shape": (1024, 1024, 128), "desc": "one z-slab of configs[4] at 8 GPUs: 1024x1024x128, f1,f2 ~ "
                                                 "U{1..10}, face x=0 -> face x=1023, M = M_bind (DRAM-resident state)"},
    "C4": {"shape": None, "desc": "configs[3]: Theorem-2 fractal omega_k, k = 10 (t = 1024), V = [-t,t]x[0,t+1], "
                                  "A = x-axis, B = (0,t), f1 in {1,2}, f2 = 1, M = infinity"},
}
for _side in (50, 75, 100, 125):   # the §6 protocol: water on the boundary, B = centre
    WORKLOADS[f"P6-{_side}"] = {"shape": (_side,) * 3, "desc": f"§6 cube {_side}^3, boundary -> centre, "
                                                             f"f1,f2 ~ U{{1..10}}, M = M_bind"}
    WORKLOADS[f"P6-{_side}-inf"] = {"shape": (_side,) * 3, "desc": f"§6 cube {_side}^3, boundary -> centre, "
                                                                 f"f1 ~ U{{1..10}}, M = infinity"}
MBIND = os.path.join(ROOT, "tests", "golden", "mbind.json")
PROFILE_SUMMARY = os.path.join(ROOT, "profiles", "roofline_traffic.json")


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def workload_instance(name: str, seed: int):
    from paper_1511_06441_b200 import instances as I
    if name == "C4":
        inst = I.fractal_instance(10)
        return inst, {"seed": 0, "F1_lex": 1024, "M_bind": I.M_INF}
    table = json.load(open(MBIND))
    if name.startswith("P6-"):
        base = name[:-4] if name.endswith("-inf") else name
        meta = dict(table[f"{base}/0"])
        M = I.M_INF if name.endswith("-inf") else meta["M_bind"]
        return I.grid_instance(WORKLOADS[name]["shape"], 0, 1, 10, "boundary", "centre", M, name), meta
    key = f"{name}/{seed}"
    if key not in table:
        key = f"{name}/0"
    M = table[key]["M_bind"]
    seed = table[key]["seed"]
    return I.config_face(WORKLOADS[name]["shape"], seed, M, name=name), table[key]


def share_nccl_id(rank: int) -> bytes:
    """NCCL unique id of the multi-GPU slab engine: made on rank 0, shared
    through torch.distributed (any backend)."""
    import torch.distributed as dist
    from paper_1511_06441_b200 import wcsp
    obj = [wcsp.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def reduce_timing(total_ms: float, units: float, device: str):
    """(max over ranks of the device time, sum over ranks of the work)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([total_ms], dtype=torch.float64, device=device)
    u = torch.tensor([float(units)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())


def alg_bytes(r, d: int) -> int:
    """Algorithmic bytes per solve: SURVEY §8(d) 'alg', per cycle
        2 (E + P) + 13 R + (2d*8 + 22) T + 8 C + 2 RL
    summed over the solve's cycles = the same formula on the solve's totals:
    2 B per live lane/phantom per cycle (u8 residual read + write), 13 B per
    arrival (L(src) 2, f2 1, L(D) 2, temp atomic 8), 2d*8 + 22 B per triggered
    vertex (neighbour label + temp, f1/f2, own lane word r/w, label write, list
    read), 8 B per phantom created, 2 B per relabel.  E + P = edge_updates,
    R = arrivals, T = triggered, C = phantoms_created, RL = relabels."""
    return (2 * r.edge_updates + 13 * r.arrivals + (2 * d * 8 + 22) * r.triggered + 8 * r.phantoms_created
            + 2 * r.relabels)


def wheel_bytes(r, d: int) -> int:
    """The timing-wheel engine's own byte model (events are not
    touched between creation and arrival): 8 B written per event created, 8 B
    read + 8 B temp read-modify-write per arrival, (24 + 2d*8) B per triggered
    vertex, 4 B per relabel.  Reported beside the §8(d) numerator."""
    return (8 * (r.lanes_started + r.phantoms_created) + 16 * r.arrivals + (24 + 2 * d * 8) * r.triggered
            + 4 * r.relabels)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for n, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def host_cpu():
    """(nproc, CPU model) of this host."""
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count(), model


def sample_instance(workload: str, side: int):
    """A bounded sample of the workload: the same recipe (value distribution, A/B
    rule, dimension, budget rule) on a cube of `side`; M_bind by the oracle's
    tier 3 (two lexicographic Dijkstras, SURVEY §8 notation)."""
    from paper_1511_06441_b200 import instances as I
    import oracle
    if workload == "C4":
        k = max(3, min(10, side.bit_length() - 1))
        return I.fractal_instance(k), f"Theorem-2 fractal k = {k} (t = {1 << k}), M = infinity"
    d = len(WORKLOADS[workload]["shape"])
    shape = (side,) * d
    if workload.startswith("P6-"):
        inst = I.grid_instance(shape, 0, 1, 10, "boundary", "centre", I.M_INF, workload)
        if workload.endswith("-inf"):
            return inst, f"{'x'.join(map(str, shape))} cube of the §6 recipe, M = infinity"
    else:
        inst = I.config_face(shape, 0, I.M_INF, name=workload)
    Mb = oracle.m_bind(inst)
    return inst.with_M(Mb), f"{'x'.join(map(str, shape))} grid of the {workload} recipe (seed 0, M_bind = {Mb})"


SIDES = {2: [64, 96, 128, 192, 256, 384, 512], 3: [24, 32, 40, 48, 56, 64, 72, 80, 96]}


def pick_side(workload: str, target_s: float) -> int:
    """The largest sample side whose tier-5 solve is predicted to take at most
    target_s (calibrated on the smallest; cost ~ N * cycles ~ side^(d+1))."""
    import oracle
    d = 2 if workload in ("C2", "C4") else 3
    sides = SIDES[d]
    inst, _ = sample_instance(workload, sides[0])
    t0 = time.perf_counter()
    oracle.solve_model(inst)
    dt0 = max(time.perf_counter() - t0, 1e-3)
    side = sides[0]
    for s_ in sides[1:]:
        if dt0 * (s_ / sides[0]) ** (d + 1) <= target_s:
            side = s_
    return side


def cpu_sample(workload: str, target_s: float):
    """The CPU baseline: oracle tier 5 — the paper's nine-step cycle run
    sequentially on one host core (oracle/wcsp_oracle.c orc_model, as it stands)
    — solving a bounded sample of the workload in full: the same recipe on the
    largest cube predicted to take at most target_s.  Its work counter is the
    metric's numerator by the same definition (sum over cycles of live edges +
    live phantoms; equal to the GPU's counters bit for bit where both run), so
    value = work / CPU seconds is directly comparable with `value`."""
    import oracle
    inst, what = sample_instance(workload, pick_side(workload, target_s))
    t0 = time.perf_counter()
    r, c = oracle.solve_model(inst)
    dt = time.perf_counter() - t0
    nproc, model = host_cpu()
    return {"value": c.work / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"oracle tier 5 (the paper's cycle run sequentially, oracle/wcsp_oracle.c orc_model) solving "
                      f"the {what} in full: {c.work} edge-updates over {c.cycles} cycles in {dt:.2f} s",
            "seconds": round(dt, 3), "host_nproc": nproc, "host_cpu": model}


def cpu_full(inst):
    """The oracle's time to solution on the bench instance itself (tier 2, one
    core, in full); run in a child process concurrently with the GPU steps
    (--cpu-full; about 6-10 minutes on C3)."""
    import oracle
    t0 = time.perf_counter()
    o = oracle.solve_pruned(inst)
    return {"tier": 2, "seconds": round(time.perf_counter() - t0, 2), "key": list(o.key()), "cores": 1}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (tier 5, as it stands) on the host cores,
    each step one bounded sample of the workload (see cpu_sample), sized so the
    whole W + K run stays within about three minutes."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    per_step = min(args.ref_seconds, 150.0 / max(1, args.warmup + args.steps))
    inst, what = sample_instance(args.workload, pick_side(args.workload, per_step))
    times, work = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        _, c = oracle.solve_model(inst)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            work.append(c.work)
    value = sum(work) / sum(times)
    nproc, model = host_cpu()
    sample = (f"oracle tier 5 (the paper's cycle run sequentially, one core) solving the {what} in full per step "
              f"({work[0]} edge-updates); host {nproc} cores, {model}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": {"workload": args.workload, "desc": WORKLOADS[args.workload]["desc"],
                                            "sample": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run
    with N ranks (rendezvous on 127.0.0.1) and return its exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C3", choices=sorted(WORKLOADS))
    ap.add_argument("--engine", default="wheel", choices=["persistent", "stepped", "wheel", "wheel_stepped"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--cpu-full", action="store_true",
                    help="also time the oracle (tier 2) solving the bench instance in full, concurrently")
    ap.add_argument("--ref-seconds", type=float, default=15.0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--partition", default="slabs", choices=["replicas", "slabs"],
                    help="N > 1: one instance cut into N z-slabs (strong scaling, default) or an independent "
                         "seed per rank (weak scaling)")
    ap.add_argument("--halo", default="peer", choices=["copy", "peer"],
                    help="slab boundary: fused over peer memory in one kernel (peer) or ghost-plane copies")
    ap.add_argument("--vslabs", type=int, default=0,
                    help="N = 1: cut the instance into this many virtual slabs on the one GPU")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args)
    if world != args.gpus and not (args.impl == "reference" and "WORLD_SIZE" not in os.environ):
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE = {world} (launch one rank per GPU)\n")
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


def run_ours(args, rank, world, local):
    import torch
    slabs = world > 1 and args.partition == "slabs"
    if world > 1:
        # NCCL's communicator lines (rank, nranks, transport) for the record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1511_06441_b200 import wcsp

    stream = torch.cuda.current_stream()
    shape = WORKLOADS[args.workload]["shape"]
    on_device = (shape is not None and int(np.prod(shape)) >= (1 << 27) and not slabs and args.vslabs <= 1
                 and not args.cpu_full)
    face = args.workload in ("C2", "C3", "C3s", "C5", "C5z8")
    if slabs and face:
        # slab partition: every rank generates ONLY its planes (slab + ghost planes) in HBM and
        # passes them with local_slab (no rank ever holds the whole grid; include/wcsp.h)
        meta = json.load(open(MBIND))[f"{args.workload}/0"]
        z0, z1, p0, p1 = wcsp.slab_planes(shape[-1], world, rank)
        f1, f2 = wcsp.generate_grid(shape, meta["seed"], 1, 10, p0, p1, stream=stream)
        A = wcsp.generate_mask(shape, "face0", p0, p1, stream=stream)
        B = wcsp.generate_mask(shape, "face1", p0, p1, stream=stream)
        torch.cuda.synchronize()
        from types import SimpleNamespace
        inst = SimpleNamespace(shape=tuple(shape), M=meta["M_bind"], name=args.workload)
        solver = wcsp.Solver(shape=shape, f1=f1, f2=f2, maskA=A, maskB=B, M=inst.M, engine="wheel", stream=stream,
                             nranks=world, rank=rank, nccl_id=share_nccl_id(rank), halo=args.halo, local_slab=True)
        del f1, f2, A, B
    elif on_device:
        # 2^27+ vertices: generate the instance in HBM (wcsp_generate_grid, the same recipe as
        # instances.grid_values) instead of building GBs of host arrays
        meta = json.load(open(MBIND))[f"{args.workload}/0"]
        f1, f2 = wcsp.generate_grid(shape, meta["seed"], 1, 10, stream=stream)
        A, B = wcsp.generate_mask(shape, "face0", stream=stream), wcsp.generate_mask(shape, "face1", stream=stream)
        from types import SimpleNamespace
        inst = SimpleNamespace(shape=tuple(shape), M=meta["M_bind"], name=args.workload)
        solver = wcsp.Solver(shape=shape, f1=f1, f2=f2, maskA=A, maskB=B, M=inst.M, engine=args.engine,
                             stream=stream)
        args.e2e_steps = 0
    else:
        inst, meta = workload_instance(args.workload, 0 if slabs else rank)
    d = len(inst.shape)
    if on_device or (slabs and face):
        pass
    elif slabs:   # one instance, slab `rank` of `world` on this GPU
        solver = wcsp.Solver(inst, engine="wheel", stream=stream, nranks=world, rank=rank,
                             nccl_id=share_nccl_id(rank), halo=args.halo)
    elif args.vslabs > 1:
        solver = wcsp.Solver(inst, engine="wheel", stream=stream, slabs=args.vslabs, halo=args.halo)
    else:
        solver = wcsp.Solver(inst, engine=args.engine, stream=stream)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > L2 (126 MB)

    full = None
    if args.cpu_full and rank == 0:          # the oracle's full solve runs beside the GPU steps
        import multiprocessing as mpc
        full = mpc.get_context("fork").Pool(1)
        full_res = full.apply_async(cpu_full, (inst,))

    for _ in range(args.warmup):
        solver.solve()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # timed region: K solves, L2 flushed between steps (outside the events)
    results = []
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            results.append(solver.solve())
            ev[i][1].record(stream)
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    updates = sum(r.edge_updates for r in results)
    if world > 1:
        # slabs: every rank reports the whole instance's (summed) work; count it once
        total_ms, updates_all = reduce_timing(total_ms, updates / world if slabs else updates, "cuda")
    else:
        updates_all = updates
    value = updates_all / (total_ms / 1000.0)

    # roofline of the dominant kernel (the persistent cycle kernel; one launch per solve)
    r0 = results[0]
    cyc_ms = statistics.mean(r.cycle_ms for r in results)
    ab = alg_bytes(r0, d)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = ab / (cyc_ms / 1000.0) / 1e9
    traffic, dram_src = None, None
    if os.path.exists(PROFILE_SUMMARY):
        try:
            ps = json.load(open(PROFILE_SUMMARY)).get(f"{args.workload}/{args.engine}")
            if ps:
                traffic, dram_src = ps["dram_bytes_per_launch"], ps.get("source")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": {"persistent": "k_persistent<D>", "wheel": "k_wheel_hybrid<D,B> (k_wheel_persistent<D> if WCSP_HYBRID=0 or ineligible)"}.get(
                    args.engine, "k_*<D> (stepped: 3 launches per cycle)") + " (cycle kernel)",
                "alg_bytes_per_launch": ab,
                "alg_formula": "SURVEY §8(d): 2(E+P) + 13R + (2d*8+22)T + 8C + 2RL over the solve's counters",
                "wheel_model_bytes_per_launch": wheel_bytes(r0, d),
                "wheel_model_gbs": round(wheel_bytes(r0, d) / (cyc_ms / 1000.0) / 1e9, 2),
                "dram_gbs": round(traffic / (cyc_ms / 1000.0) / 1e9, 2) if traffic else None,
                "dram_source": dram_src,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback B200_PROFILING.md 6.65 TB/s"}

    # e2e through the C-ABI with host buffers (pinned): H2D of the step's inputs + solve + result read
    e2e = None
    if args.e2e_steps > 0 and not slabs and args.vslabs <= 1:
        pin = {k: torch.from_numpy(np.ascontiguousarray(getattr(inst, k))).pin_memory()
               for k in ("f1", "f2", "maskA", "maskB")}
        host = {k: v.numpy() for k, v in pin.items()}
        h2d = sum(v.numel() for v in pin.values())
        e_ms, e_upd = [], 0
        barrier()
        for i in range(args.e2e_steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            solver.load(f1=host["f1"], f2=host["f2"], maskA=host["maskA"], maskB=host["maskB"], M=inst.M)
            rr = solver.solve()
            b.record(stream)
            b.synchronize()
            e_ms.append(a.elapsed_time(b))
            e_upd += rr.edge_updates
        et = sum(e_ms)
        if world > 1:
            et, e_upd = reduce_timing(et, e_upd / world if slabs else e_upd, "cuda")
        e2e = {"value": e_upd / (et / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": 5760, "ms_per_step": et / args.e2e_steps,
               "path": "wcsp_load (pinned host f1,f2,A,B -> HBM, validate, weight build) + wcsp_solve + result "
                       "D2H (the 5760-byte control block, sizeof(Ctl))"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_sample(args.workload, args.cpu_seconds)
    cpu_full_rec = None
    if full is None and args.workload in ("C3", "C2", "C3s"):
        # not timed in this run (22 min on C3): the recorded time to solution of the same instance by
        # the oracle's tier 2, with where it was measured; `--cpu-full` times it beside the GPU steps
        gold = os.path.join(ROOT, "tests", "golden", "tier2_full.json")
        rec = json.load(open(gold)).get(f"{args.workload}/0") if os.path.exists(gold) else None
        box = os.path.join(ROOT, "profiles", "r02", "bench_cpu_full_r02x.jsonl")
        secs, where = (rec or {}).get("cpu_seconds"), "tests/golden/tier2_full.json (dev host, 1 core)"
        if args.workload == "C3" and os.path.exists(box):
            try:
                secs = json.loads(open(box).readline())["cpu_full"]["seconds"]
                where = "profiles/r02/bench_cpu_full_r02x.jsonl (a B200 box's host, 1 core, --cpu-full)"
            except Exception:
                pass
        if rec and secs:
            cpu_full_rec = {"tier": 2, "seconds": secs, "key": rec["key"], "cores": 1,
                            "recorded": where + "; not timed in this run (--cpu-full times it beside the GPU steps)",
                            "matches_gpu": rec["key"] == list(results[0].key()),
                            "gpu_speedup_time_to_solution": round(secs * 1000.0 / (total_ms / args.steps), 1)}
    if full is not None:
        cpu_full_rec = full_res.get()
        cpu_full_rec["matches_gpu"] = cpu_full_rec["key"] == list(r0.key())
        cpu_full_rec["gpu_speedup_time_to_solution"] = round(cpu_full_rec["seconds"] * 1000.0 / (total_ms / args.steps), 1)
        full.close()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if slabs else "weak", "vs_baseline": None, "dtype": "u16", "data": "synthetic",
            "config": {"workload": args.workload, "desc": WORKLOADS[args.workload]["desc"],
                       "shape": list(inst.shape), "seed": meta["seed"], "M": inst.M,
                       "M_bind_from": "tests/golden/mbind.json (oracle, scripts/make_mbind.py)",
                       "engine": args.engine, "l2": "flushed between steps (256 MiB write outside the events)",
                       "parallelism": (f"{world} z-slabs of one instance ("
                                       + ("boundary fused over NVLink peer memory, one kernel per GPU"
                                          if args.halo == "peer" else "NCCL send/recv + allreduce per cycle") + ")"
                                       if slabs else f"{world} independent instances (one seed per rank)")
                                      if world > 1 else (f"1 GPU, {args.vslabs} virtual z-slabs ({args.halo} halo)"
                                                         if args.vslabs > 1 else "1 GPU")},
            "solve_ms": total_ms / args.steps,
            "solve": {"F1": r0.F1, "F2": r0.F2, "X": r0.X, "Y": r0.Y, "cycles": r0.cycles,
                      "edge_updates": r0.edge_updates, "arrivals": r0.arrivals, "triggered": r0.triggered,
                      "phantoms_created": r0.phantoms_created, "relabels": r0.relabels,
                      "lanes_started": r0.lanes_started, "peak_phantoms": r0.peak_phantoms,
                      "cycle_ms": r0.cycle_ms, "device_ms": r0.device_ms, "retries": r0.retries},
            "hbm_gbs_alg": round(achieved, 2),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "cpu_full": cpu_full_rec,
            "e2e": e2e,
            "gpu_launches": int(sum(r.kernel_launches for r in results)),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    solver.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main() or 0)
