"""Benchmark of the FED-FEM explicit step (BASELINE.json metric: element-steps/s,
ms/step, % of HBM roofline).

Default workload: BASELINE config 4 -- the >=10M-element temperature-dependent
mesh named by north_star's roofline target (256^3 trilinear hexes, 16.8M
elements, 16.97M nodes, TD k/c/perfusion, per-element log-normal conductivity
factor, moving Gaussian source, Dirichlet 37 C on all faces, fp32), one fused
step kernel per step.  ``--config cfg1|cfg2|cfg3`` selects another workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fast|reference]

Timing: W warm-up steps, then K steps bracketed by a barrier +
synchronize, CUDA events on the engine's stream, max over ranks.  The
per-step input (1.1 GB of slot + node streams for cfg4) is larger than the
126 MB L2, so no L2 flush is needed between steps.  ``e2e`` is the same metric
through the public C ABI with host buffers (pinned host T in, one step,
host T out, every step; on one GPU fh_step_host_async double-buffers the
host I/O so step k's download overlaps step k+1's upload).  ``--impl reference`` times the CPU oracle
(restated reference path, oracle/fh_oracle.c, all host threads) on the same
full workload (same mesh, boundary, sources, dt), one oracle step per bench
step, and (cfg4) the unmodified numba reference from baseline/_ref on the
largest cube its chunk buffers fit (128^3), labelled as such.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fast", choices=["fast", "reference"])
    ap.add_argument("--config", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--precision", type=int, default=0)
    ap.add_argument("--divisions", type=int, default=0, help="override mesh divisions (testing)")
    ap.add_argument("--part-nodes", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--numba-divisions", type=int, default=128,
                    help="reference arm, cfg4: also time the unmodified numba reference on this cube (0: skip)")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def make_problem(name, divisions=0, precision=0):
    from paper_1909_05098_b200 import configs

    fn = getattr(configs, name)
    kw = {}
    if divisions:
        kw["scale" if name == "cfg5" else "divisions"] = divisions
    if precision and name in ("cfg2", "cfg3"):
        kw["precision"] = precision
    prob = fn(**kw)
    if precision:
        prob.precision = precision
    return prob


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.samples = []
        self.proc = None
        self.index = index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu=timestamp,{self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [s for ts, s in self.samples if t0 - 0.05 <= ts <= t1 + 0.05] or [s for _, s in self.samples[-3:]]
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            parts = [p.strip() for p in r.split(",")]
            try:
                sm.append(float(parts[1]))
                smax = max(smax, float(parts[2]))
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_for(prob):
    """The CPU oracle (restated reference path, oracle/fh_oracle.c) on `prob`'s
    full mesh and boundary, with the dt the GPU arm uses (0.9 x Gershgorin)."""
    from oracle import oracle as orc
    from paper_1909_05098_b200.solver import resolve_boundary
    from paper_1909_05098_b200.sources import robin_lumps

    mesh = prob.mesh
    rb = resolve_boundary(prob.boundary, mesh)
    robin = robin_lumps(mesh, prob.robin[0], exclude=rb.dirichlet_nodes) if prob.robin else None
    def model(sources):
        return orc.OracleModel(mesh, prob.materials or prob.material,
                               dirichlet=(rb.dirichlet_nodes, rb.dirichlet_values),
                               sources=[s.as_dict() for s in sources], robin=robin, kfactor=prob.kfactor,
                               elem_region=prob.element_region, td_mode=prob.td_mode)

    ora = model(prob.sources)
    dt = 0.9 * ora.critical_dt(np.full(mesh.n_nodes, 37.0))
    if prob.name == "cfg4":  # the moving source of the fast arm depends on dt (run_sources)
        del ora
        ora = model(run_sources(prob, dt))
    ora.initial_state(37.0)
    return ora, dt, orc.max_threads()


def run_sources(prob, dt):
    """cfg4's moving Gaussian covers its seeded segment over the run's steps."""
    import paper_1909_05098_b200 as fh

    a, b = (np.asarray(v) for v in prob.notes["path"])
    return [fh.GaussianSource(amp=5.0e6, sigma=0.005, x0=tuple(a), vel=tuple((b - a) / (prob.steps * dt)), t0=0.0)]


def oracle_step_times(ora, dt, steps):
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        ora.step(dt, 1)
        times.append(time.perf_counter() - t0)
    return times


def numba_reference_rate(divisions, steps):
    """The UNMODIFIED reference (fedheat, numba, baseline/_ref) through its own
    public API on the largest cfg4-family cube its O(E*V) chunk buffers allow on
    the host: TD laws of cfg2, Dirichlet 37 C on every
    face, all host threads.  The reference has no k-factor or moving source."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "fedheat")):
        return {"unavailable": "baseline/_ref not installed"}
    code = f"""
import json, os, sys, time
sys.path.insert(0, {ref!r})
import numpy as np
import fedheat as fh
mesh = fh.generate_cube_mesh("hex", {divisions}, 0.1)
lin = lambda y0, s: fh.PropertyCurve(temperatures=np.array([0.0, 2000.0]), values=np.array([y0 * (1 + s * (0 - 37)), y0 * (1 + s * (2000 - 37))]))
mat = fh.TissueMaterial(density=fh.PropertyCurve(temperatures=np.array([0.0]), values=np.array([1060.0])), specific_heat=lin(3600.0, -0.0005),
                        conductivity=lin(0.5, 0.0013), perfusion_rate=0.525, blood_specific_heat=3640.0,
                        arterial_temperature=37.0, metabolic_rate=420.0)
bnd = fh.BoundarySpec(dirichlet=tuple((f, 37.0) for f in ("x0", "x1", "y0", "y1", "z0", "z1")))
eng = fh.ExplicitEngine(mesh, mat, bnd)
nw = os.cpu_count()
eng.run(37.0, steps=2, auto_dt_safety=0.9, workers=nw)  # numba compile + buffers
res = eng.run(37.0, steps={steps}, auto_dt_safety=0.9, workers=nw)
print(json.dumps({{"per_step_s": res.timings["per_step_s"], "elements": mesh.n_elements, "workers": res.workers}}))
"""
    env = dict(os.environ)
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/fh_numba_cache")
    env["NUMBA_NUM_THREADS"] = str(os.cpu_count())
    try:
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900, env=env)
        d = json.loads(out.stdout.strip().splitlines()[-1])
    except Exception as ex:  # noqa: BLE001
        err = (out.stderr.strip().splitlines() or [""])[-1] if "out" in locals() else ""
        return {"unavailable": f"reference run failed: {type(ex).__name__} {err}"[:300]}
    return {"value": d["elements"] / d["per_step_s"], "unit": "element-steps/s", "cores": d["workers"],
            "kind": "reference", "sample": f"fedheat (numba, unmodified, baseline/_ref) ExplicitEngine.run on a "
            f"{divisions}^3 hex cube ({d['elements']} elements), TD cfg2 laws, {steps} steps after a 2-step warm-up "
            f"(timings per_step_s); the full cfg4 needs n_chunks x V x 8 B = 556 GB of reference chunk buffers"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # the FULL workload of the fast arm (same mesh, boundary, extensions and dt),
    # one oracle step per bench step on all host threads
    prob = make_problem(args.config, args.divisions, args.precision)
    t0 = time.perf_counter()
    ora, dt, threads = oracle_for(prob)
    setup = time.perf_counter() - t0
    times = oracle_step_times(ora, dt, args.warmup + args.steps)
    per_step = times[args.warmup:]
    tot = sum(per_step)
    elem = prob.mesh.n_elements
    value = elem * len(per_step) / tot
    sample = (f"full {args.config} workload ({elem} elements, the fast arm's mesh, boundary, sources and dt), one "
              f"oracle step (oracle/fh_oracle.c: the reference's operation order restated in C, fp64, OpenMP on "
              f"{threads} threads of {cpu_model()}) per bench step")
    line = {
        "impl": "reference", "metric": "element-steps/sec", "value": value, "unit": "element-steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(per_step),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "elements": elem, "nodes": prob.mesh.n_nodes,
                   "same_config": args.divisions == 0,
                   "dt_s": dt, "oracle_setup_s": setup, "cpu": cpu_model()},
        "cpu_baseline": {"value": value, "unit": "element-steps/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "element-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.config == "cfg4" and args.numba_divisions > 0:
        line["reference_numba"] = numba_reference_rate(args.numba_divisions, 3)
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch

    import paper_1909_05098_b200 as fh
    from paper_1909_05098_b200 import _native as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prob = make_problem(args.config, args.divisions, args.precision)
    mesh = prob.mesh
    t_setup = time.perf_counter()
    if world > 1:
        from paper_1909_05098_b200.dist import make_engine

        # cfg4 is slab-partitioned along z (BASELINE.json); 8 domains so that the
        # tiles -- and therefore the results -- are the same for 1/2/4/8 GPUs
        eng = make_engine(mesh, prob.material, prob.boundary, rank=rank, world=world, device=local,
                          n_domains=8, slab_axis=2 if prob.name == "cfg4" else -1, part_nodes=args.part_nodes,
                          **prob.engine_kwargs())
    elif prob.name in ("cfg1", "cfg2") and prob.precision == 64:
        # small fp64 configs: the reference-exact EXACT engine, whose resident
        # kernel runs the whole step loop in one cooperative launch
        eng = fh.ExplicitEngine(mesh, prob.material, prob.boundary, assembly="exact", device=local,
                                **prob.engine_kwargs())
    else:  # same tiles as the multi-GPU runs: one engine owning all 8 domains
        eng = fh.ExplicitEngine(mesh, prob.material, prob.boundary, assembly="tiled", device=local,
                                part_nodes=args.part_nodes, n_domains=8,
                                slab_axis=2 if prob.name == "cfg4" else -1, **prob.engine_kwargs())
    t_setup = time.perf_counter() - t_setup
    dt = 0.9 * eng.critical_dt(37.0)
    if prob.name == "cfg4":  # moving source: traverse the seeded segment over the run
        eng.set_sources(run_sources(prob, dt))
    st = eng.initial_state(37.0)
    import ctypes as C

    L, h = eng._L, eng._h
    T = st.temperatures
    N.check(L.fh_set_temperature(h, N.ptr(T), T.size, 0, 0.0))
    stream = torch.cuda.ExternalStream(eng.stream())
    rep = N.FhReport()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    # warm-up right before the timed region (no idle gap for the clocks to drop)
    N.check(L.fh_step(h, args.warmup, dt, C.byref(rep)))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    L2_BYTES = 126 * 2**20
    flush_l2 = eng.layout()["step_bytes"] < 2 * L2_BYTES
    resident = eng.layout()["kernels_per_step"] == 0
    wall0 = time.time()
    elapsed = C.c_float(0.0)
    if resident:
        # the resident EXACT kernel: the K steps are one cooperative launch
        # (the step loop of solver.py:468-493 on the device); L2 is flushed
        # (2x-L2 buffer overwritten) right before it
        scratch = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=f"cuda:{local}")
        scratch.fill_(1)
        rc = L.fh_step_timed(h, args.steps, dt, C.byref(rep), C.byref(elapsed))
    elif not flush_l2:
        # CUDA events recorded on the engine's launch stream around the K launches
        rc = L.fh_step_timed(h, args.steps, dt, C.byref(rep), C.byref(elapsed))
    else:
        # the step's working set fits in L2: a 2x-L2 buffer is overwritten on
        # the engine stream before every step and each step is timed alone
        scratch = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=f"cuda:{local}")
        rc = L.fh_step_timed_flush(h, args.steps, dt, C.c_void_p(scratch.data_ptr()), scratch.numel(),
                                   C.byref(rep), C.byref(elapsed))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall1 = time.time()
    N.check(rc)
    del stream
    ms_total = float(elapsed.value)
    if world > 1:  # max over ranks
        t = torch.tensor([ms_total], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    time.sleep(0.15)
    sampler.stop()
    clocks = sampler.summary(wall0, wall1)
    lay = eng.layout()
    E = mesh.n_elements
    ms = ms_total / args.steps
    value = E * args.steps / (ms_total / 1e3)
    peak, peak_kind = peaks()
    # per GPU: the canonical bytes of this GPU's share of the mesh
    achieved = lay["canonical_bytes"] / world / (ms / 1e3) / 1e9
    # e2e: through the public C ABI with pinned host buffers, one step per call
    # (the full fp64 field goes host->device and back every step, on every
    # rank).  One GPU: fh_step_host_async double-buffers the host I/O, so the
    # upload of step k+1 and the download of step k use both bus directions
    # at once; N > 1: the synchronous fh_step_host.
    Tin = torch.empty(mesh.n_nodes, dtype=torch.float64, pin_memory=True)
    Touts = [torch.empty(mesh.n_nodes, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    Tin.numpy()[:] = T
    p_in = C.cast(C.c_void_p(Tin.data_ptr()), N.f64p)
    p_out = [C.cast(C.c_void_p(t.data_ptr()), N.f64p) for t in Touts]
    K = args.e2e_steps
    if world == 1:
        for q in (0, 1):  # warm both slots (buffers, streams, events)
            N.check(L.fh_step_host_async(h, p_in, p_out[q], T.size, 1, dt, q))
            N.check(L.fh_host_wait(h, q, C.byref(rep)))
        t0 = time.perf_counter()
        for k in range(K):
            N.check(L.fh_step_host_async(h, p_in, p_out[k % 2], T.size, 1, dt, k % 2))
            if k >= 1:
                N.check(L.fh_host_wait(h, (k - 1) % 2, C.byref(rep)))
        N.check(L.fh_host_wait(h, (K - 1) % 2, C.byref(rep)))
        e2e_s = (time.perf_counter() - t0) / K
    else:
        N.check(L.fh_step_host(h, p_in, p_out[0], T.size, 1, dt, C.byref(rep)))
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(K):
            N.check(L.fh_step_host(h, p_in, p_out[0], T.size, 1, dt, C.byref(rep)))
        e2e_s = (time.perf_counter() - t0) / K
    if world > 1:
        t = torch.tensor([e2e_s], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    traffic = None  # ncu DRAM bytes of this config's step kernel(s) at this precision
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and not resident:
        with open(tpath) as f:
            traffic = json.load(f).get(f"{args.config}_f{prob.precision}")
    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        # bounded sample: the oracle on the same full mesh, 1 warm-up + n steps
        ora, odt, threads = oracle_for(prob)
        n = 3 if E > 1e6 else 50
        ts = oracle_step_times(ora, odt, 1 + n)[1:]
        del ora
        cpu = {"value": E * n / sum(ts), "unit": "element-steps/s", "cores": threads, "kind": "port",
               "sample": f"oracle (fh_oracle.c, fp64, reference op order, OpenMP, {cpu_model()}) on the full "
                         f"{args.config} mesh ({E} elements), {n} steps after 1 warm-up"}
    line = {
        "metric": "element-steps/sec", "value": value, "unit": "element-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if prob.precision == 32 else "f64",
        "data": "synthetic (seeded, BASELINE.json shapes)",
        "config": {"workload": prob.name, "elements": E, "nodes": mesh.n_nodes, "td": prob.td_mode,
                   "assembly": "exact (resident: %d steps per launch, %d CTAs)" % (args.steps, lay["resident_ctas"])
                   if resident else "tiled", "parts": lay["n_parts"], "slots": lay["n_slots"],
                   "parallelism": f"{world} GPU domain decomposition (8 z-slab domains, NCCL halo exchange)"
                   if world > 1 else "1 GPU",
                   "l2": ("working set < 2x L2: 252 MB buffer overwritten before the timed launch (the K steps "
                          "run in one launch; between steps the mesh stays L2/shared-memory resident by design)"
                          if resident else
                          "working set < 2x L2: 252 MB buffer overwritten before every timed step" if flush_l2
                          else "per-step input > 2x 126 MB L2 (no flush needed)"), "dt_s": dt, "setup_s": t_setup},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_kind": peak_kind,
                     "canonical_bytes_per_step": lay["canonical_bytes"], "layout_bytes_per_step": lay["step_bytes"]},
        "cpu_baseline": cpu,
        "e2e": {"value": E / e2e_s, "unit": "element-steps/s", "h2d_bytes_per_step": 8 * mesh.n_nodes,
                "d2h_bytes_per_step": 8 * mesh.n_nodes},
        # step kernel launches (one per tile kind and launch range) + halo pack / unpack (N > 1)
        # (resident: one launch for all K steps)
        "gpu_launches": 1 if resident else args.steps * (lay["kernels_per_step"] + (2 if world > 1 else 0)),
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        del eng
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
