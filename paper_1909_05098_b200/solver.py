"""Explicit FED-FEM time stepping on the B200 (reference API, GPU engine).

Public surface of /root/reference/pkg/src/fedheat/solver.py:53-564 --
`PackedElements`, `BoundarySpec`, `resolve_boundary`, `SimState`,
`RunResult`, `element_conductivity`, `element_loads`, `scatter_loads`,
`ExplicitEngine` (initial_state / step / critical_dt / run),
`run_simulation`, `critical_dt` -- with the same argument meaning, error types
and step semantics:

  * TD mode refreshes k(T), kbar_e and C(T) every step; constant mode freezes
    them at the first step after `initial_state` (solver.py:280-303);
  * heat loads are active on [t0, t1) at the step-start time (solver.py:307-318);
  * Dirichlet values are imposed after every update (solver.py:364-365);
  * a non-finite or |T| > runaway_limit field raises InstabilityError(step,
    time, node) with the node = first non-finite, else argmax |T| (:369-382);
  * time = step_index * dt (:366-367).

Every step runs on the GPU through libfedheat_b200.so.  ``assembly="exact"``
(default, fp64) reproduces the reference bit for bit; ``assembly="tiled"`` is
the fused single-kernel step (fp64 or fp32) for large meshes.  Extensions
(keyword-only, parity unpinned): volumetric ``sources``, ``robin``
conditions, per-element ``kfactor``, material ``regions``.
"""

from __future__ import annotations

import ctypes as C
import logging
import math
import time as _time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from . import kernels
from .element import ElemKind, ElementPrecomp, batch_precompute
from .errors import ConfigError, InstabilityError
from .material import TissueMaterial, eval_property
from .mesh import Mesh
from .precompute import lumped_from_volumes, lumped_mass
from .sources import RobinSpec, robin_lumps, static_nodal_power

log = logging.getLogger(__name__)

CHUNK_SIZE = N.CHUNK_SIZE
DEFAULT_RUNAWAY_LIMIT = 1.0e6
DEFAULT_DT_RECHECK = 100


class PackedElements:
    """Flat element arrays in the reference layout (solver.py:53-88).

    conn_data/conn_offs: node ids per element (tets then hexes); mat_data/
    mat_offs: row-major A per element; row_abs: |A| row sums; volumes.
    Host-side arrays (numpy precompute, same bits as the reference); the
    chunk scratch ``buffers`` of the reference is not materialised.
    """

    def __init__(self, mesh: Mesh):
        counts, conn, mats, rowabs, vols = [], [], [], [], []
        for kind, c in ((ElemKind.TET4, mesh.tets), (ElemKind.HEX8, mesh.hexes)):
            if c.shape[0] == 0:
                continue
            a, vol = batch_precompute(kind, mesh.nodes[c])
            counts.append(np.full(c.shape[0], kind.n_nodes, dtype=np.int64))
            conn.append(c.ravel())
            mats.append(a.reshape(-1))
            rowabs.append(np.abs(a).sum(axis=2).ravel())
            vols.append(vol)
        counts = np.concatenate(counts)
        self.n_nodes = mesh.n_nodes
        self.n_elements = int(counts.size)
        self.node_counts = counts
        self.conn_offs = np.concatenate(([0], np.cumsum(counts))).astype(np.int64)
        self.conn_data = np.concatenate(conn).astype(np.int64)
        self.mat_offs = np.concatenate(([0], np.cumsum(counts * counts))).astype(np.int64)
        self.mat_data = np.concatenate(mats)
        self.row_abs = np.concatenate(rowabs)
        self.volumes = np.concatenate(vols)
        self.n_chunks = -(-self.n_elements // CHUNK_SIZE)


@dataclass(frozen=True)
class BoundarySpec:
    """Named-set boundary conditions (solver.py:91-102).

    dirichlet: (set, T) pairs imposed after every step; heat_loads: (set,
    watts per node, t_start, t_end), active while t_start <= t < t_end.
    """

    dirichlet: tuple = ()
    heat_loads: tuple = ()


@dataclass(frozen=True)
class ResolvedBoundary:
    dirichlet_nodes: np.ndarray
    dirichlet_values: np.ndarray
    loads: tuple

    def apply_dirichlet(self, temperatures) -> np.ndarray:
        out = np.array(temperatures, dtype=np.float64)
        out[self.dirichlet_nodes] = self.dirichlet_values
        return out


def resolve_boundary(boundary: BoundarySpec, mesh: Mesh) -> ResolvedBoundary:
    """Node sets -> sorted Dirichlet ids/values and load lists (solver.py:118-164)."""

    def members(name):
        if name not in mesh.node_sets:
            known = ", ".join(sorted(mesh.node_sets)) or "<none>"
            raise ConfigError(f"mesh has no node set {name!r} (available: {known})")
        return mesh.node_sets[name]

    fixed: dict[int, float] = {}
    for name, value in boundary.dirichlet:
        value = float(value)
        if not math.isfinite(value):
            raise ConfigError(f"non-finite Dirichlet value on set {name!r}")
        for node in members(name).tolist():
            prev = fixed.get(node)
            if prev is not None and prev != value:
                raise ConfigError(f"node {node} has conflicting Dirichlet values ({prev} and {value})")
            fixed.setdefault(node, value)
    loads = []
    for name, power, t0, t1 in boundary.heat_loads:
        power, t0, t1 = float(power), float(t0), float(t1)
        if not (math.isfinite(power) and math.isfinite(t0) and math.isfinite(t1)):
            raise ConfigError(f"non-finite heat-load parameters on set {name!r}")
        if t1 <= t0:
            raise ConfigError(f"heat load on set {name!r} has empty window [{t0}, {t1})")
        loads.append((members(name), power, t0, t1))
    ids = np.fromiter(fixed.keys(), dtype=np.int64, count=len(fixed))
    vals = np.fromiter(fixed.values(), dtype=np.float64, count=len(fixed))
    order = np.argsort(ids, kind="stable")
    return ResolvedBoundary(dirichlet_nodes=ids[order], dirichlet_values=vals[order], loads=tuple(loads))


@dataclass
class SimState:
    temperatures: np.ndarray
    time: float = 0.0
    step_index: int = 0
    inflow: np.ndarray = field(init=False)

    def __post_init__(self):
        self.temperatures = np.ascontiguousarray(self.temperatures, dtype=np.float64)
        self.inflow = np.zeros_like(self.temperatures)


@dataclass
class RunResult:
    state: SimState
    dt: float
    n_steps: int
    dt_critical: float
    td_mode: bool
    workers: int
    probe_nodes: np.ndarray
    probe_times: np.ndarray
    probe_values: np.ndarray
    timings: dict


def element_conductivity(material: TissueMaterial, temperatures, node_ids) -> float:
    """Mean nodal conductivity of one element, sequential sum (kernels.py:89-98)."""
    total, count = 0.0, 0
    for nid in node_ids:
        total += eval_property(material.conductivity, float(temperatures[nid]))
        count += 1
    return total / count


def element_loads(precomp: ElementPrecomp, kbar: float, t_local) -> np.ndarray:
    """kbar * A @ (T_local - T_local[0]) for one element (outflow positive)."""
    a = precomp.unit_conductance
    n = a.shape[0]
    base = float(t_local[0])
    out = np.empty(n)
    for r in range(n):
        acc = 0.0
        for b in range(n):
            acc += a[r, b] * (float(t_local[b]) - base)
        out[r] = kbar * acc
    return out


def scatter_loads(packed: PackedElements, kbar, temperatures, out=None) -> np.ndarray:
    """Net conduction inflow per node on the GPU (chunked order, == reference bitwise)."""
    if out is None:
        out = np.empty(packed.n_nodes)
    kernels.scatter_net_loads(packed.conn_data, packed.conn_offs, packed.mat_data, packed.mat_offs, kbar,
                              temperatures, packed.n_chunks, CHUNK_SIZE, None, out)
    return out


def _curve(cv, keep):
    if cv is None:
        return N.FhCurve(0, None, None)
    x, y = N.f64(cv.temperatures), N.f64(cv.values)
    if x.size > N.MAX_KNOTS:
        raise ConfigError(f"property curves are limited to {N.MAX_KNOTS} knots on the GPU")
    keep += [x, y]
    return N.FhCurve(x.size, N.ptr(x), N.ptr(y))


def _source_array(sources):
    arr = (N.FhSource * max(1, len(sources)))()
    for i, s in enumerate(sources):
        d = s.as_dict()
        arr[i] = N.FhSource(0 if d["kind"] == "gauss" else 1, d["amp"], d["sigma"], d["cap"],
                            (C.c_double * 3)(*d["x0"]), (C.c_double * 3)(*d["vel"]), d["t0"], d["t1"])
    return arr


def native_inputs(mesh, bnd, materials, *, sources=(), robin=(), kfactor=None, element_region=None,
                  td_mode=False, precision=64, assembly="exact", runaway_limit=DEFAULT_RUNAWAY_LIMIT, device=0,
                  part_nodes=0, n_domains=1, domains=None, slab_axis=-1, tuning=None):
    """C-ABI descriptors (fh_mesh, fh_boundary, fh_options) for a problem.

    Returns (mesh, boundary, options, keep, robin) -- ``keep`` holds the numpy
    arrays the descriptors point into; it must outlive every native call.
    """
    keep = []
    nodes, tets, hexes = N.f64(mesh.nodes), N.i64(mesh.tets), N.i64(mesh.hexes)
    keep += [nodes, tets, hexes]
    fm = N.FhMesh(mesh.n_nodes, N.ptr(nodes), tets.shape[0], N.ptr(tets, N.i64p), hexes.shape[0],
                  N.ptr(hexes, N.i64p))
    fb = N.FhBoundary()
    dn, dv = N.i64(bnd.dirichlet_nodes), N.f64(bnd.dirichlet_values)
    keep += [dn, dv]
    fb.n_dirichlet, fb.dirichlet_nodes, fb.dirichlet_values = dn.size, N.ptr(dn, N.i64p), N.ptr(dv)
    if bnd.loads:
        offs = np.zeros(len(bnd.loads) + 1, np.int64)
        for i, ld in enumerate(bnd.loads):
            offs[i + 1] = offs[i] + ld[0].size
        lnodes = N.i64(np.concatenate([ld[0] for ld in bnd.loads]))
        lp = N.f64([ld[1] for ld in bnd.loads])
        l0 = N.f64([ld[2] for ld in bnd.loads])
        l1 = N.f64([ld[3] for ld in bnd.loads])
        keep += [offs, lnodes, lp, l0, l1]
        fb.n_loads, fb.load_offsets, fb.load_nodes = len(bnd.loads), N.ptr(offs, N.i64p), N.ptr(lnodes, N.i64p)
        fb.load_power, fb.load_t0, fb.load_t1 = N.ptr(lp), N.ptr(l0), N.ptr(l1)
    dyn = [s for s in sources if not s.is_static]
    if dyn:
        arr = _source_array(dyn)
        keep.append(arr)
        fb.n_sources, fb.sources = len(dyn), C.cast(arr, C.POINTER(N.FhSource))
    robin_out = None
    robin = tuple(robin) if isinstance(robin, (list, tuple)) else (robin,)
    if robin:
        parts = [robin_lumps(mesh, r, exclude=bnd.dirichlet_nodes) for r in robin if isinstance(r, RobinSpec)]
        rn = np.concatenate([p[0] for p in parts])
        ra = np.concatenate([p[1] for p in parts])
        rb = np.concatenate([p[2] for p in parts])
        if np.unique(rn).size != rn.size:
            raise ConfigError("a node is in more than one Robin set")
        rn, ra, rb = N.i64(rn), N.f64(ra), N.f64(rb)
        keep += [rn, ra, rb]
        robin_out = (rn, ra, rb)
        fb.n_robin, fb.robin_nodes, fb.robin_hA, fb.robin_hAT = rn.size, N.ptr(rn, N.i64p), N.ptr(ra), N.ptr(rb)
    mats = (N.FhMaterial * len(materials))()
    for r, m in enumerate(materials):
        mats[r] = N.FhMaterial(_curve(m.density, keep), _curve(m.specific_heat, keep), _curve(m.conductivity, keep),
                               _curve(m.perfusion_curve, keep), m.perfusion_rate, m.blood_specific_heat,
                               m.arterial_temperature, m.metabolic_rate)
    keep.append(mats)
    fo = N.FhOptions()
    fo.precision, fo.assembly, fo.td_mode, fo.device = int(precision), N.ASSEMBLY[assembly], int(td_mode), int(device)
    fo.runaway_limit = float(runaway_limit)
    fo.n_materials, fo.materials = len(materials), C.cast(mats, C.POINTER(N.FhMaterial))
    if element_region is not None:
        er = np.ascontiguousarray(element_region, dtype=np.int32)
        keep.append(er)
        fo.element_region = N.ptr(er, N.i32p)
    if kfactor is not None:
        kf = N.f64(kfactor)
        keep.append(kf)
        fo.element_kfactor = N.ptr(kf)
    fo.part_nodes = int(part_nodes)
    fo.n_domains = int(n_domains)
    lo, hi = domains if domains is not None else (0, int(n_domains))
    fo.domain_lo, fo.domain_hi, fo.slab_axis = int(lo), int(hi), int(slab_axis)
    for name, value in (tuning or {}).items():
        if name not in N.TUNING_FIELDS:
            raise ConfigError(f"unknown tuning knob {name!r} (known: {', '.join(N.TUNING_FIELDS)})")
        setattr(fo, name, int(value))
    return fm, fb, fo, keep, robin_out


class ExplicitEngine:
    """GPU-resident explicit engine for one model (solver.py:243-519)."""

    def __init__(self, mesh: Mesh, material: TissueMaterial, boundary: BoundarySpec | None = None, *,
                 td_mode: bool | None = None, runaway_limit: float = DEFAULT_RUNAWAY_LIMIT,
                 dt_recheck_interval: int = DEFAULT_DT_RECHECK, precision: int = 64, assembly: str = "exact",
                 sources=(), robin=(), kfactor=None, materials=None, element_region=None, device: int = 0,
                 part_nodes: int = 0, n_domains: int = 1, domains=None, slab_axis: int = -1, tuning=None):
        t_begin = _time.perf_counter()
        self.mesh = mesh
        self.material = material
        self.materials = list(materials) if materials is not None else [material]
        self.boundary = resolve_boundary(boundary or BoundarySpec(), mesh)
        self.td_mode = (not all(m.is_constant for m in self.materials)) if td_mode is None else bool(td_mode)
        self.runaway_limit = float(runaway_limit)
        self.dt_recheck_interval = int(dt_recheck_interval)
        if self.dt_recheck_interval < 1:
            raise ConfigError("dt_recheck_interval must be >= 1")
        if assembly not in N.ASSEMBLY:
            raise ConfigError(f"unknown assembly {assembly!r}")
        if precision not in (32, 64):
            raise ConfigError("precision must be 32 or 64")
        self.precision = int(precision)
        self.assembly = assembly
        self.sources = tuple(sources)
        self._packed = None
        self._inflow_kept = False
        N.require_gpu()
        fm, fb, fo, keep, self.robin = native_inputs(
            mesh, self.boundary, self.materials, sources=self.sources, robin=robin, kfactor=kfactor,
            element_region=element_region, td_mode=self.td_mode, precision=self.precision, assembly=assembly,
            runaway_limit=self.runaway_limit, device=device, part_nodes=part_nodes, n_domains=n_domains,
            domains=domains, slab_axis=slab_axis, tuning=tuning)
        self._keep = keep
        self._h = None
        handle = C.c_void_p()
        N.check(N.lib().fh_create(C.byref(fm), C.byref(fb), C.byref(fo), C.byref(handle)))
        self._h = handle
        # static sources are lumped with the device-computed volumes: Q(x_i) * v_i
        static = [s for s in self.sources if s.is_static]
        self.q_static = None
        if static:
            vols = np.empty(mesh.n_nodes)
            N.check(N.lib().fh_get_precompute(handle, N.ptr(vols), None))
            self.q_static = N.f64(static_nodal_power(static, mesh.nodes, vols))
            N.check(N.lib().fh_set_q_static(handle, N.ptr(self.q_static), mesh.n_nodes))
        self._L = N.lib()
        vols = np.empty(mesh.n_nodes)
        N.check(self._L.fh_get_precompute(self._h, N.ptr(vols), None))
        self.lumped = lumped_from_volumes(vols, material)
        self.precompute_seconds = _time.perf_counter() - t_begin

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.fh_destroy(h)
            self._h = None

    # -- device state / multi-domain helpers ------------------------------------
    def temperature(self) -> np.ndarray:
        """Current device field (original numbering, float64)."""
        T = np.empty(self.n_nodes)
        N.check(self._L.fh_get_temperature(self._h, N.ptr(T), T.size))
        return T

    def owned_mask(self) -> np.ndarray:
        m = np.zeros(self.n_nodes, np.uint8)
        N.check(self._L.fh_get_owned(self._h, m.ctypes.data_as(C.POINTER(C.c_uint8)), m.size))
        return m.astype(bool)

    def halo_info(self) -> dict:
        w, r, npeer = C.c_int32(), C.c_int32(), C.c_int32()
        ns, nr, nb, nparts = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        N.check(self._L.fh_halo_info(self._h, C.byref(w), C.byref(r), C.byref(npeer), C.byref(ns), C.byref(nr),
                                     C.byref(nb), C.byref(nparts)))
        return {"world": w.value, "rank": r.value, "n_peers": npeer.value, "n_send": ns.value,
                "n_recv": nr.value, "boundary_parts": nb.value, "parts": nparts.value}

    def halo_lists(self):
        i = self.halo_info()
        peers = np.empty(i["n_peers"], np.int32)
        so, ro = np.empty(i["n_peers"] + 1, np.int64), np.empty(i["n_peers"] + 1, np.int64)
        sn, rn = np.empty(i["n_send"], np.int64), np.empty(i["n_recv"], np.int64)
        N.check(self._L.fh_halo_lists(self._h, N.ptr(peers, N.i32p), N.ptr(so, N.i64p), N.ptr(sn, N.i64p),
                                      N.ptr(ro, N.i64p), N.ptr(rn, N.i64p)))
        return peers, so, sn, ro, rn

    def halo_export(self) -> np.ndarray:
        out = np.empty(self.halo_info()["n_send"])
        N.check(self._L.fh_halo_export(self._h, N.ptr(out)))
        return out

    def halo_import(self, values) -> None:
        v = N.f64(values)
        N.check(self._L.fh_halo_import(self._h, N.ptr(v)))

    def set_sources(self, sources) -> None:
        """Replace the time-dependent sources (static ones stay folded into q_static)."""
        dyn = [s for s in sources if not s.is_static]
        arr = _source_array(dyn)
        N.check(self._L.fh_set_sources(self._h, C.cast(arr, C.POINTER(N.FhSource)), len(dyn)))
        self.sources = tuple(s for s in self.sources if s.is_static) + tuple(dyn)

    @property
    def packed(self) -> PackedElements:
        if self._packed is None:
            self._packed = PackedElements(self.mesh)
        return self._packed

    @property
    def n_nodes(self) -> int:
        return self.mesh.n_nodes

    def layout(self) -> dict:
        lay = N.FhLayout()
        N.check(self._L.fh_get_layout(self._h, C.byref(lay)))
        return {k: getattr(lay, k) for k, _ in N.FhLayout._fields_}

    def stream(self) -> int:
        return int(self._L.fh_stream(self._h) or 0)

    # -- state ---------------------------------------------------------------
    def initial_state(self, initial_temperature) -> SimState:
        t0 = np.asarray(initial_temperature, dtype=np.float64)
        if t0.ndim == 0:
            t0 = np.full(self.n_nodes, float(t0))
        if t0.shape != (self.n_nodes,):
            raise ConfigError(f"initial field has shape {t0.shape}, expected ({self.n_nodes},)")
        if not np.isfinite(t0).all():
            raise ConfigError("initial field contains non-finite temperatures")
        state = SimState(temperatures=t0.copy())
        bnd = self.boundary
        state.temperatures[bnd.dirichlet_nodes] = bnd.dirichlet_values
        cap = lumped_mass(self.material, self.lumped.node_volumes, state.temperatures)
        free = np.ones(self.n_nodes, dtype=bool)
        free[bnd.dirichlet_nodes] = False
        if np.any(cap[free] <= 0.0):
            bad = int(np.argmax(free & (cap <= 0.0)))
            raise ConfigError(f"node {bad} has zero heat capacity (outside every element?) "
                              "but is not Dirichlet-constrained")
        N.check(self._L.fh_reset_properties(self._h))
        return state

    def _raise_instability(self, state: SimState, rep) -> None:
        node = int(rep.fail_node)
        val = state.temperatures[node]
        what = "non-finite" if not np.isfinite(val) else f"{val:.3g} C"
        raise InstabilityError(f"temperature at node {node} is {what}; the step size likely exceeds the stable limit",
                               step=state.step_index, time=state.time, node=node)

    def step(self, state: SimState, dt: float) -> None:
        """Advance one explicit step in place (host state in, host state out)."""
        T = state.temperatures
        if T.dtype != np.float64 or not T.flags.c_contiguous:
            raise ConfigError("state.temperatures must be a contiguous float64 array")
        # one upload (fh_set_temperature: field + clock), the step, one download
        N.check(self._L.fh_set_temperature(self._h, N.ptr(T), T.size, int(state.step_index), float(state.time)))
        if self.assembly != "exact" and not self._inflow_kept:
            N.check(self._L.fh_keep_inflow(self._h, 1))  # TILED: the step kernel also writes F
            self._inflow_kept = True
        rep = N.FhReport()
        rc = self._L.fh_step_host(self._h, None, N.ptr(T), T.size, 1, float(dt), C.byref(rep))
        state.step_index = int(rep.step_index)
        state.time = float(rep.time)
        # state.inflow = this step's F (solver.py:352); TILED: 0 at Dirichlet nodes
        N.check(self._L.fh_get_inflow(self._h, N.ptr(state.inflow), T.size))
        if rc == 2:
            self._raise_instability(state, rep)
        N.check(rc)

    def critical_dt(self, temperatures) -> float:
        """Gershgorin bound 2/lambda_hat (solver.py:384-405), bitwise == reference."""
        t = np.asarray(temperatures, dtype=np.float64)
        if t.ndim == 0:
            t = np.full(self.n_nodes, float(t))
        t = N.f64(t)
        out = C.c_double()
        N.check(self._L.fh_critical_dt(self._h, N.ptr(t), t.size, C.byref(out)))
        return float(out.value)

    def critical_dt_current(self) -> float:
        out = C.c_double()
        N.check(self._L.fh_critical_dt(self._h, None, self.n_nodes, C.byref(out)))
        return float(out.value)

    # -- run -----------------------------------------------------------------
    def run(self, initial_temperature, *, steps: int, dt: float | None = None,
            auto_dt_safety: float | None = None, workers: int | None = None, probes=None,
            probe_interval: int = 1, snapshot_interval: int = 0, on_snapshot=None) -> RunResult:
        if steps < 1:
            raise ConfigError(f"steps must be >= 1, got {steps}")
        if (dt is None) == (auto_dt_safety is None):
            raise ConfigError("give exactly one of dt or auto_dt_safety")
        if probe_interval < 1 or snapshot_interval < 0:
            raise ConfigError("probe_interval must be >= 1 and snapshot_interval >= 0")
        applied = kernels.set_workers(workers if workers else kernels.default_workers())
        state = self.initial_state(initial_temperature)
        dt_cr = self.critical_dt(state.temperatures)
        if auto_dt_safety is not None:
            if not (0.0 < auto_dt_safety <= 1.0):
                raise ConfigError(f"auto_dt_safety must be in (0, 1], got {auto_dt_safety}")
            if not math.isfinite(dt_cr):
                raise ConfigError("cannot auto-pick dt: the critical step is unbounded")
            dt = auto_dt_safety * dt_cr
        dt = float(dt)
        if not (dt > 0.0 and math.isfinite(dt)):
            raise ConfigError(f"dt must be positive and finite, got {dt}")
        if dt > dt_cr:
            log.warning("dt = %.6g s exceeds the estimated critical step %.6g s; the run may go unstable", dt, dt_cr)
        probe_nodes = np.asarray([] if probes is None else probes, dtype=np.int64)
        if probe_nodes.size and (probe_nodes.min() < 0 or probe_nodes.max() >= self.n_nodes):
            raise ConfigError("probe node index out of range")
        T = state.temperatures
        N.check(self._L.fh_set_temperature(self._h, N.ptr(T), T.size, 0, 0.0))
        cap = steps // probe_interval
        N.check(self._L.fh_set_probes(self._h, N.ptr(probe_nodes, N.i64p), probe_nodes.size, probe_interval, cap))
        first_row = T[probe_nodes].copy()
        if on_snapshot is not None and snapshot_interval > 0:
            on_snapshot(state)
        # segment boundaries: TD dt rechecks and snapshots need the host in the loop
        stops = {steps}
        if self.td_mode:
            stops.update(range(self.dt_recheck_interval, steps, self.dt_recheck_interval))
        if on_snapshot is not None and snapshot_interval > 0:
            stops.update(range(snapshot_interval, steps, snapshot_interval))
        dt_exceeds = dt > dt_cr
        rep = N.FhReport()
        t_begin = _time.perf_counter()
        done = 0
        for stop in sorted(stops):
            if self.td_mode and done > 0 and done % self.dt_recheck_interval == 0:
                now = self.critical_dt_current()
                if dt > now and not dt_exceeds:
                    log.warning("dt = %.6g s has crossed above the critical step (now %.6g s) at step %d",
                                dt, now, done)
                dt_exceeds = dt > now
            rc = self._L.fh_step(self._h, stop - done, dt, C.byref(rep))
            done = int(rep.step_index)
            if rc == 2:
                N.check(self._L.fh_get_temperature(self._h, N.ptr(T), T.size))
                state.step_index, state.time = done, float(rep.time)
                self._raise_instability(state, rep)
            N.check(rc)
            if on_snapshot is not None and snapshot_interval > 0 and done % snapshot_interval == 0 and done < steps:
                N.check(self._L.fh_get_temperature(self._h, N.ptr(T), T.size))
                state.step_index, state.time = done, float(rep.time)
                on_snapshot(state)
        N.check(self._L.fh_get_temperature(self._h, N.ptr(T), T.size))
        stepping = _time.perf_counter() - t_begin
        state.step_index, state.time = done, float(rep.time)
        if self.assembly == "exact" or self._inflow_kept:
            N.check(self._L.fh_get_inflow(self._h, N.ptr(state.inflow), T.size))
        if on_snapshot is not None:
            on_snapshot(state)
        rows = np.empty((cap, probe_nodes.size))
        nrec = C.c_int64()
        N.check(self._L.fh_get_probes(self._h, N.ptr(rows), cap, C.byref(nrec)))
        values = np.vstack([first_row[None, :], rows[: nrec.value]]) if probe_nodes.size else \
            np.empty((1 + steps // probe_interval, 0))
        times = np.array([0.0] + [k * probe_interval * dt for k in range(1, 1 + steps // probe_interval)])
        # the reference records state.time = step_index * dt
        times[1:] = np.array([(k * probe_interval) * dt for k in range(1, 1 + steps // probe_interval)])
        return RunResult(state=state, dt=dt, n_steps=steps, dt_critical=dt_cr, td_mode=self.td_mode,
                         workers=applied, probe_nodes=probe_nodes, probe_times=times, probe_values=values,
                         timings={"precompute_s": self.precompute_seconds, "stepping_s": stepping,
                                  "per_step_s": stepping / steps})


def run_simulation(mesh: Mesh, material: TissueMaterial, boundary: BoundarySpec | None = None, *,
                   initial_temperature, steps: int, dt: float | None = None, auto_dt_safety: float | None = None,
                   td_mode: bool | None = None, workers: int | None = None, probes=None, probe_interval: int = 1,
                   snapshot_interval: int = 0, on_snapshot=None, runaway_limit: float = DEFAULT_RUNAWAY_LIMIT,
                   dt_recheck_interval: int = DEFAULT_DT_RECHECK, **engine_kwargs) -> RunResult:
    engine = ExplicitEngine(mesh, material, boundary, td_mode=td_mode, runaway_limit=runaway_limit,
                            dt_recheck_interval=dt_recheck_interval, **engine_kwargs)
    return engine.run(initial_temperature, steps=steps, dt=dt, auto_dt_safety=auto_dt_safety, workers=workers,
                      probes=probes, probe_interval=probe_interval, snapshot_interval=snapshot_interval,
                      on_snapshot=on_snapshot)


def critical_dt(mesh: Mesh, material: TissueMaterial, temperatures) -> float:
    return ExplicitEngine(mesh, material).critical_dt(temperatures)
