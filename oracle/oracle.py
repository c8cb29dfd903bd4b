"""ctypes front end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Used by tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs -- never by the product package.  The C code
restates the reference step (/root/reference/pkg/src/fedheat/kernels.py:61-142,
solver.py:280-405, element.py:69-171, precompute.py:43-62, mesh.py:128-150);
its parity is pinned bit for bit to the reference by tests/test_oracle_golden.py
against tests/golden/*.npz (made by tests/golden/make_golden.py, which runs
the reference package itself).

Inputs are duck-typed: anything with ``nodes/tets/hexes`` (mesh) and the
reference's ``TissueMaterial`` attributes works, so the same call accepts the
reference's own objects and this repo's.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

CHUNK = 4096

f64p = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)


class OcCurve(C.Structure):
    _fields_ = [("n", C.c_int32), ("x", f64p), ("y", f64p)]


class OcMat(C.Structure):
    _fields_ = [("rho", OcCurve), ("c", OcCurve), ("k", OcCurve), ("wb", OcCurve),
                ("wb_const", C.c_double), ("cb", C.c_double), ("Ta", C.c_double), ("Qm", C.c_double)]


class OcSource(C.Structure):
    _fields_ = [("kind", C.c_int32), ("amp", C.c_double), ("sigma", C.c_double), ("cap", C.c_double),
                ("x0", C.c_double * 3), ("vel", C.c_double * 3), ("t0", C.c_double), ("t1", C.c_double)]


class OcConfig(C.Structure):
    _fields_ = [
        ("V", C.c_int64), ("xyz", f64p), ("n_tet", C.c_int64), ("tets", i64p),
        ("n_hex", C.c_int64), ("hexes", i64p), ("n_mat", C.c_int32), ("mats", C.POINTER(OcMat)),
        ("elem_region", i32p), ("kfactor", f64p), ("n_dir", C.c_int64), ("dir_nodes", i64p),
        ("dir_vals", f64p), ("n_robin", C.c_int64), ("robin_nodes", i64p), ("robin_hA", f64p),
        ("robin_hAT", f64p), ("n_loads", C.c_int64), ("load_offs", i64p), ("load_nodes", i64p),
        ("load_power", f64p), ("load_t0", f64p), ("load_t1", f64p), ("q_static", f64p),
        ("n_src", C.c_int32), ("srcs", C.POINTER(OcSource)), ("td_mode", C.c_int32),
        ("runaway_limit", C.c_double),
    ]


def build() -> str:
    """Compile liboracle.so (gcc, -ffp-contract=off) if missing or stale."""
    src = os.path.join(_HERE, "fh_oracle.c")
    if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.oc_create.restype = C.c_void_p
        L.oc_create.argtypes = [C.POINTER(OcConfig), C.c_char_p, C.c_int]
        L.oc_destroy.argtypes = [C.c_void_p]
        L.oc_set_state.argtypes = [C.c_void_p, f64p, C.c_int64, C.c_double]
        L.oc_get_state.argtypes = [C.c_void_p, f64p, i64p, f64p]
        L.oc_step.argtypes = [C.c_void_p, C.c_double, C.c_int64, i64p, i64p]
        L.oc_run_probes.argtypes = [C.c_void_p, C.c_double, C.c_int64, i64p, C.c_int64, C.c_int64,
                                    f64p, i64p, i64p, i64p]
        L.oc_scatter.argtypes = [C.c_void_p, f64p, f64p, f64p]
        L.oc_critical_dt.restype = C.c_double
        L.oc_critical_dt.argtypes = [C.c_void_p, f64p]
        L.oc_get_precompute.argtypes = [C.c_void_p, f64p, f64p, f64p, f64p]
        L.oc_get_inflow.argtypes = [C.c_void_p, f64p]
        L.oc_get_csr.argtypes = [C.c_void_p, i64p, i64p]
        L.oc_set_threads.argtypes = [C.c_int]
        L.oc_max_threads.restype = C.c_int
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().oc_set_threads(int(n))


def max_threads() -> int:
    return int(lib().oc_max_threads())


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _curve(cv, keep):
    if cv is None:
        return OcCurve(0, None, None)
    x = np.ascontiguousarray(cv.temperatures, dtype=np.float64)
    y = np.ascontiguousarray(cv.values, dtype=np.float64)
    keep += [x, y]
    return OcCurve(x.size, _p(x, f64p), _p(y, f64p))


class InstabilityInOracle(Exception):
    def __init__(self, step, node):
        self.step, self.node = int(step), int(node)
        super().__init__(f"oracle instability at step {step}, node {node}")


class OracleModel:
    """One oracle model.

    mesh        : object with nodes (V,3), tets (Et,4), hexes (Eh,8)
    materials   : a TissueMaterial-like object, or a list of them (regions)
    dirichlet   : (node ids, values) sorted unique, or None
    loads       : list of (node ids, power, t0, t1), reference heat_loads semantics
    q_static    : (V,) static extra nodal power (W), e.g. lumped volumetric sources
    sources     : list of dicts {kind: "gauss"|"rf", amp, sigma, cap, x0, vel, t0, t1}
    robin       : (node ids, hA, hA*Tinf) or None
    kfactor     : (E,) per-element conductivity factor or None
    elem_region : (E,) region index per element or None
    """

    def __init__(self, mesh, materials, *, dirichlet=None, loads=(), q_static=None, sources=(),
                 robin=None, kfactor=None, elem_region=None, td_mode=None, runaway_limit=1.0e6):
        L = lib()
        keep = []
        self._keep = keep
        mats = list(materials) if isinstance(materials, (list, tuple)) else [materials]
        nodes = np.ascontiguousarray(mesh.nodes, dtype=np.float64)
        tets = np.ascontiguousarray(np.asarray(mesh.tets, dtype=np.int64).reshape(-1, 4))
        hexes = np.ascontiguousarray(np.asarray(mesh.hexes, dtype=np.int64).reshape(-1, 8))
        keep += [nodes, tets, hexes]
        self.V = nodes.shape[0]
        self.E = tets.shape[0] + hexes.shape[0]
        self.nconn = 4 * tets.shape[0] + 8 * hexes.shape[0]
        self.n_tet = tets.shape[0]
        omats = (OcMat * len(mats))()
        td = False
        for r, m in enumerate(mats):
            pc = getattr(m, "perfusion_curve", None)
            omats[r] = OcMat(_curve(m.density, keep), _curve(m.specific_heat, keep),
                             _curve(m.conductivity, keep), _curve(pc, keep),
                             float(m.perfusion_rate), float(m.blood_specific_heat),
                             float(m.arterial_temperature), float(m.metabolic_rate))
            td = td or (not m.is_constant)
        keep.append(omats)
        self.td_mode = td if td_mode is None else bool(td_mode)
        cfg = OcConfig()
        cfg.V, cfg.xyz = self.V, _p(nodes, f64p)
        cfg.n_tet, cfg.tets = tets.shape[0], _p(tets, i64p)
        cfg.n_hex, cfg.hexes = hexes.shape[0], _p(hexes, i64p)
        cfg.n_mat, cfg.mats = len(mats), C.cast(omats, C.POINTER(OcMat))
        if elem_region is not None:
            er = np.ascontiguousarray(elem_region, dtype=np.int32)
            keep.append(er)
            cfg.elem_region = _p(er, i32p)
        if kfactor is not None:
            kf = np.ascontiguousarray(kfactor, dtype=np.float64)
            keep.append(kf)
            cfg.kfactor = _p(kf, f64p)
        if dirichlet is not None and len(dirichlet[0]):
            dn = np.ascontiguousarray(dirichlet[0], dtype=np.int64)
            dv = np.ascontiguousarray(dirichlet[1], dtype=np.float64)
            keep += [dn, dv]
            cfg.n_dir, cfg.dir_nodes, cfg.dir_vals = dn.size, _p(dn, i64p), _p(dv, f64p)
            self.dirichlet = (dn, dv)
        else:
            self.dirichlet = (np.empty(0, np.int64), np.empty(0))
        if robin is not None and len(robin[0]):
            rn = np.ascontiguousarray(robin[0], dtype=np.int64)
            ra = np.ascontiguousarray(robin[1], dtype=np.float64)
            rb = np.ascontiguousarray(robin[2], dtype=np.float64)
            keep += [rn, ra, rb]
            cfg.n_robin, cfg.robin_nodes, cfg.robin_hA, cfg.robin_hAT = rn.size, _p(rn, i64p), _p(ra, f64p), _p(rb, f64p)
        loads = list(loads)
        if loads:
            offs = np.zeros(len(loads) + 1, dtype=np.int64)
            for i, ld in enumerate(loads):
                offs[i + 1] = offs[i] + len(ld[0])
            lnodes = np.ascontiguousarray(np.concatenate([np.asarray(ld[0], np.int64) for ld in loads]))
            pw = np.array([ld[1] for ld in loads], dtype=np.float64)
            t0 = np.array([ld[2] for ld in loads], dtype=np.float64)
            t1 = np.array([ld[3] for ld in loads], dtype=np.float64)
            keep += [offs, lnodes, pw, t0, t1]
            cfg.n_loads, cfg.load_offs, cfg.load_nodes = len(loads), _p(offs, i64p), _p(lnodes, i64p)
            cfg.load_power, cfg.load_t0, cfg.load_t1 = _p(pw, f64p), _p(t0, f64p), _p(t1, f64p)
        if q_static is not None:
            qs = np.ascontiguousarray(q_static, dtype=np.float64)
            keep.append(qs)
            cfg.q_static = _p(qs, f64p)
        sources = list(sources)
        if sources:
            arr = (OcSource * len(sources))()
            for i, s in enumerate(sources):
                arr[i] = OcSource(0 if s["kind"] == "gauss" else 1, float(s.get("amp", 0.0)),
                                  float(s.get("sigma", 1.0)), float(s.get("cap", math.inf)),
                                  (C.c_double * 3)(*s.get("x0", (0, 0, 0))),
                                  (C.c_double * 3)(*s.get("vel", (0, 0, 0))),
                                  float(s.get("t0", -math.inf)), float(s.get("t1", math.inf)))
            keep.append(arr)
            cfg.n_src, cfg.srcs = len(sources), C.cast(arr, C.POINTER(OcSource))
        cfg.td_mode = int(self.td_mode)
        cfg.runaway_limit = float(runaway_limit)
        err = C.create_string_buffer(256)
        h = L.oc_create(C.byref(cfg), err, 256)
        if not h:
            raise ValueError(err.value.decode())
        self._h = C.c_void_p(h)
        self._L = L

    def __del__(self):
        if getattr(self, "_h", None) is not None:
            self._L.oc_destroy(self._h)
            self._h = None

    # -- precompute -------------------------------------------------------
    def precompute(self):
        nA = 16 * self.n_tet + 64 * (self.E - self.n_tet)
        A, vol = np.empty(nA), np.empty(self.E)
        ra, nv = np.empty(self.nconn), np.empty(self.V)
        self._L.oc_get_precompute(self._h, _p(A, f64p), _p(vol, f64p), _p(ra, f64p), _p(nv, f64p))
        return {"mat_data": A, "volumes": vol, "row_abs": ra, "node_volumes": nv}

    def csr(self):
        offs, pos = np.empty(self.V + 1, np.int64), np.empty(self.nconn, np.int64)
        self._L.oc_get_csr(self._h, _p(offs, i64p), _p(pos, i64p))
        return offs, pos

    # -- state / stepping -------------------------------------------------
    def set_state(self, T, step_index=0, time=0.0):
        T = np.ascontiguousarray(np.broadcast_to(np.asarray(T, np.float64), (self.V,)))
        self._L.oc_set_state(self._h, _p(T, f64p), int(step_index), float(time))

    def initial_state(self, T0):
        T = np.array(np.broadcast_to(np.asarray(T0, np.float64), (self.V,)))
        dn, dv = self.dirichlet
        T[dn] = dv
        self.set_state(T, 0, 0.0)
        return T

    def state(self):
        T = np.empty(self.V)
        si, t = C.c_int64(), C.c_double()
        self._L.oc_get_state(self._h, _p(T, f64p), C.byref(si), C.byref(t))
        return T, int(si.value), float(t.value)

    @property
    def T(self):
        return self.state()[0]

    def inflow(self):
        out = np.empty(self.V)
        self._L.oc_get_inflow(self._h, _p(out, f64p))
        return out

    def step(self, dt, nsteps=1):
        fs, fn = C.c_int64(-1), C.c_int64(-1)
        rc = self._L.oc_step(self._h, float(dt), int(nsteps), C.byref(fs), C.byref(fn))
        if rc == 2:
            raise InstabilityInOracle(fs.value, fn.value)

    def run(self, T0, steps, dt, probes=(), interval=1):
        """initial_state + steps; returns (T, probe history incl. step 0)."""
        T = self.initial_state(T0)
        probes = np.ascontiguousarray(probes, dtype=np.int64)
        hist = np.empty((steps // interval + 1, probes.size))
        hist[0] = T[probes]
        nrec, fs, fn = C.c_int64(), C.c_int64(-1), C.c_int64(-1)
        rc = self._L.oc_run_probes(self._h, float(dt), int(steps), _p(probes, i64p), probes.size,
                                   int(interval), _p(hist[1:], f64p), C.byref(nrec), C.byref(fs), C.byref(fn))
        if rc == 2:
            raise InstabilityInOracle(fs.value, fn.value)
        return self.T, hist[: 1 + nrec.value]

    def scatter(self, kbar, T):
        kb = np.ascontiguousarray(kbar, np.float64)
        Tc = np.ascontiguousarray(T, np.float64)
        out = np.empty(self.V)
        self._L.oc_scatter(self._h, _p(kb, f64p), _p(Tc, f64p), _p(out, f64p))
        return out

    def critical_dt(self, T):
        Tc = np.ascontiguousarray(np.broadcast_to(np.asarray(T, np.float64), (self.V,)))
        return float(self._L.oc_critical_dt(self._h, _p(Tc, f64p)))
