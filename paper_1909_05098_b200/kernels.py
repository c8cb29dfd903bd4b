"""Operator layer: the reference's five kernels, executed on the GPU.

Same names, argument meaning and caller-allocated outputs as
/root/reference/pkg/src/fedheat/kernels.py:76-142; each call goes through the
C ABI (include/fedheat_b200.h, "operator layer") and is bit-identical to the
numba kernel it replaces.  ``scatter_net_loads`` keeps the chunk semantics but
ignores the reference's O(n_chunks * n_nodes) ``buffers`` scratch.

Worker control (kernels.py:33-58) is kept for API compatibility: results of
this engine never depend on it (the GPU path is deterministic by
construction); the applied count is reported back as 1.
"""

from __future__ import annotations

import os

import numpy as np

from . import _native as N
from .errors import ConfigError

_workers = 1


def max_workers() -> int:
    return max(1, int(os.environ.get("NUMBA_NUM_THREADS", "1") or 1), 1)


def set_workers(count: int) -> int:
    global _workers
    count = int(count)
    if count < 1:
        raise ConfigError(f"worker count must be >= 1, got {count}")
    _workers = min(count, max_workers())
    return _workers


def default_workers() -> int:
    env = os.environ.get("FEDHEAT_THREADS")
    if env:
        try:
            count = int(env)
        except ValueError:
            raise ConfigError(f"FEDHEAT_THREADS must be an integer, got {env!r}") from None
        if count < 1:
            raise ConfigError(f"FEDHEAT_THREADS must be >= 1, got {count}")
        return min(count, max_workers())
    return max_workers()


def warmup() -> None:
    """Load the native library (and create the CUDA context) once."""
    N.lib()
    if N.device_count() > 0:
        eval_curve_nodes(np.array([0.0, 1.0]), np.array([1.0, 2.0]), np.array([0.5]), np.empty(1))


def eval_curve_nodes(xs, ys, temps, out):
    xs, ys, t = N.f64(xs), N.f64(ys), N.f64(temps)
    res = np.empty(t.size)
    N.check(N.lib().fh_eval_curve_nodes(N.ptr(xs), N.ptr(ys), xs.size, N.ptr(t), t.size, N.ptr(res)))
    out[...] = res


def lumped_capacity_nodes(rho_x, rho_y, c_x, c_y, temps, vols, out):
    rx, ry, cx, cy = N.f64(rho_x), N.f64(rho_y), N.f64(c_x), N.f64(c_y)
    t, v = N.f64(temps), N.f64(vols)
    res = np.empty(t.size)
    N.check(N.lib().fh_lumped_capacity_nodes(N.ptr(rx), N.ptr(ry), rx.size, N.ptr(cx), N.ptr(cy), cx.size,
                                             N.ptr(t), N.ptr(v), t.size, N.ptr(res)))
    out[...] = res


def element_mean_nodal(conn_data, conn_offs, nodal, out):
    c, o, nd = N.i64(conn_data), N.i64(conn_offs), N.f64(nodal)
    res = np.empty(o.size - 1)
    N.check(N.lib().fh_element_mean_nodal(N.ptr(c, N.i64p), N.ptr(o, N.i64p), o.size - 1, N.ptr(nd), nd.size,
                                          N.ptr(res)))
    out[...] = res


def scatter_net_loads(conn_data, conn_offs, mat_data, mat_offs, kbar, temps, n_chunks, chunk_size, buffers, out):
    c, o, m, mo = N.i64(conn_data), N.i64(conn_offs), N.f64(mat_data), N.i64(mat_offs)
    kb, t = N.f64(kbar), N.f64(temps)
    res = np.empty(np.shape(out)[0])
    N.check(N.lib().fh_scatter_net_loads(N.ptr(c, N.i64p), N.ptr(o, N.i64p), N.ptr(m), N.ptr(mo, N.i64p),
                                         o.size - 1, N.ptr(kb), N.ptr(t), res.size, int(chunk_size), N.ptr(res)))
    out[...] = res


def nodal_update(temps, inflow, capacity, perf_k, perf_q, metab_q, extra_q, dt):
    t = N.f64(temps).copy()
    arrs = [N.f64(a) for a in (inflow, capacity, perf_k, perf_q, metab_q, extra_q)]
    N.check(N.lib().fh_nodal_update(N.ptr(t), *[N.ptr(a) for a in arrs], t.size, float(dt)))
    temps[...] = t
