"""Generate the golden fixtures by running the REFERENCE package itself.

Run here (the reference is mounted read-only at /root/reference; it cannot
travel to the GPU box, so its outputs are committed as small .npz fixtures):

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py

Every fixture stores its inputs (mesh arrays, material, boundary, dt, ...)
and the reference's outputs, so the tests never need /root/reference.
Reference entry points used (all /root/reference/pkg/src/fedheat/):
  solver.PackedElements (solver.py:53-88)   -> mat_data, row_abs, volumes
  precompute.build_lumped (precompute.py:43) -> node volumes, kb, qb, qm
  solver.scatter_loads (solver.py:223-240)   -> chunked scatter
  solver.ExplicitEngine.run / step / critical_dt (solver.py:322-519)
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")

import fedheat  # noqa: E402
from fedheat.errors import InstabilityError  # noqa: E402
from fedheat.mesh import Mesh  # noqa: E402
from fedheat.meshgen import generate_cube_mesh  # noqa: E402
from fedheat.material import PropertyCurve, TissueMaterial  # noqa: E402
from fedheat.precompute import build_lumped  # noqa: E402
from fedheat.scenario import load_scenario  # noqa: E402
from fedheat.solver import BoundarySpec, ExplicitEngine, PackedElements, scatter_loads  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
SCEN = os.path.join(REF, "fedheat", "scenarios")


def mat_dict(m: TissueMaterial) -> dict:
    out = {}
    for name in ("density", "specific_heat", "conductivity"):
        cv = getattr(m, name)
        out[f"mat_{name}_x"] = cv.temperatures
        out[f"mat_{name}_y"] = cv.values
    for name in ("perfusion_rate", "blood_specific_heat", "arterial_temperature", "metabolic_rate"):
        out[f"mat_{name}"] = np.float64(getattr(m, name))
    return out


def mesh_dict(mesh: Mesh) -> dict:
    return {"nodes": mesh.nodes, "tets": mesh.tets, "hexes": mesh.hexes}


def mixed_mesh(rng, div, size, jitter=0.12):
    """Jittered cube with a random tet/hex choice per cell (non-conforming is fine)."""
    from fedheat.meshgen import _HEX_OFFSETS, _TET_PATTERNS

    npts = div + 1
    axis = np.linspace(0.0, size, npts)
    zz, yy, xx = np.meshgrid(axis, axis, axis, indexing="ij")
    nodes = np.column_stack([xx.ravel(), yy.ravel(), zz.ravel()])
    nodes = nodes + rng.uniform(-jitter, jitter, nodes.shape) * (size / div)
    idx = lambda i, j, k: i + npts * (j + npts * k)  # noqa: E731
    tets, hexes = [], []
    for i in range(div):
        for j in range(div):
            for k in range(div):
                b = np.array([i, j, k])
                if rng.random() < 0.5:
                    tets += [[idx(*(b + o)) for o in p] for p in _TET_PATTERNS]
                else:
                    hexes.append([idx(*(b + o)) for o in _HEX_OFFSETS])
    return Mesh(nodes=nodes, tets=np.asarray(tets, np.int64).reshape(-1, 4),
                hexes=np.asarray(hexes, np.int64).reshape(-1, 8), node_sets={"all": np.arange(nodes.shape[0])})


def jittered(rng, kind, div, size, amount=0.2):
    base = generate_cube_mesh(kind, div, size)
    nodes = base.nodes.copy()
    interior = np.ones(base.n_nodes, bool)
    for s in ("x0", "x1", "y0", "y1", "z0", "z1"):
        interior[base.node_sets[s]] = False
    nodes[interior] += rng.uniform(-amount, amount, (interior.sum(), 3)) * (size / div)
    return Mesh(nodes=nodes, tets=base.tets, hexes=base.hexes, node_sets=base.node_sets)


def gen_precompute():
    rng = np.random.default_rng(20240101)
    for tag, mesh in (
        ("mixed3", mixed_mesh(rng, 3, 0.7)),
        ("mixed5", mixed_mesh(rng, 5, 0.05)),
        ("tet4j", jittered(rng, "tet", 4, 0.1)),
        ("hex4j", jittered(rng, "hex", 4, 0.1)),
    ):
        packed = PackedElements(mesh)
        mat = TissueMaterial.constant(density=1060.0, specific_heat=3700.0, conductivity=0.518,
                                      perfusion_rate=26.6, metabolic_rate=33800.0)
        lump = build_lumped(mesh, mat)
        np.savez_compressed(
            os.path.join(OUT, f"precompute_{tag}.npz"), **mesh_dict(mesh),
            mat_data=packed.mat_data, row_abs=packed.row_abs, volumes=packed.volumes,
            conn_data=packed.conn_data, conn_offs=packed.conn_offs,
            node_volumes=lump.node_volumes, perfusion_conductance=lump.perfusion_conductance,
            perfusion_heat=lump.perfusion_heat, metabolic_heat=lump.metabolic_heat, **mat_dict(mat))
        print("precompute", tag, packed.n_elements)


def gen_scatter():
    rng = np.random.default_rng(7)
    # > 2 chunks of 4096 elements so the chunked reduction order matters
    mesh = generate_cube_mesh("tet", 12, 0.1)
    nodes = mesh.nodes.copy()
    interior = np.ones(mesh.n_nodes, bool)
    for s in ("x0", "x1", "y0", "y1", "z0", "z1"):
        interior[mesh.node_sets[s]] = False
    nodes[interior] += rng.uniform(-0.2, 0.2, (interior.sum(), 3)) * (0.1 / 12)
    mesh = Mesh(nodes=nodes, tets=mesh.tets, hexes=mesh.hexes)
    packed = PackedElements(mesh)
    out = {}
    for r in range(3):
        T = rng.uniform(20.0, 60.0, mesh.n_nodes)
        kbar = rng.uniform(0.3, 0.8, packed.n_elements)
        out[f"T{r}"], out[f"kbar{r}"] = T, kbar
        out[f"inflow{r}"] = scatter_loads(packed, kbar, T).copy()
    np.savez_compressed(os.path.join(OUT, "scatter_tet12.npz"), **mesh_dict(mesh), **out)
    print("scatter", packed.n_elements, packed.n_chunks)


def save_run(tag, mesh, mat, boundary, T0, steps, dt=None, auto=None, td_mode=None, probes=(),
             interval=1, extra=None):
    eng = ExplicitEngine(mesh, mat, boundary, td_mode=td_mode)
    res = eng.run(T0, steps=steps, dt=dt, auto_dt_safety=auto, probes=np.asarray(probes, np.int64),
                  probe_interval=interval)
    bnd = eng.boundary
    loads_nodes = [ld[0] for ld in bnd.loads]
    d = {
        **mesh_dict(mesh), **mat_dict(mat),
        "T0": np.broadcast_to(np.asarray(T0, np.float64), (mesh.n_nodes,)).copy(),
        "steps": np.int64(steps), "dt": np.float64(res.dt), "dt_critical": np.float64(res.dt_critical),
        "td_mode": np.int64(res.td_mode), "dir_nodes": bnd.dirichlet_nodes, "dir_vals": bnd.dirichlet_values,
        "load_offs": np.concatenate([[0], np.cumsum([len(n) for n in loads_nodes])]).astype(np.int64),
        "load_nodes": (np.concatenate(loads_nodes) if loads_nodes else np.empty(0)).astype(np.int64),
        "load_power": np.array([ld[1] for ld in bnd.loads], np.float64),
        "load_t0": np.array([ld[2] for ld in bnd.loads], np.float64),
        "load_t1": np.array([ld[3] for ld in bnd.loads], np.float64),
        "probes": np.asarray(probes, np.int64), "interval": np.int64(interval),
        "T_final": res.state.temperatures, "probe_values": res.probe_values, "probe_times": res.probe_times,
        "time_final": np.float64(res.state.time),
    }
    if extra:
        d.update(extra)
    np.savez_compressed(os.path.join(OUT, f"run_{tag}.npz"), **d)
    print("run", tag, mesh.n_elements, steps, res.state.temperatures.max())


def gen_runs():
    # the bundled verification scenarios (shortened), through the public API
    for name, steps in (("conduction", 400), ("perfusion", 300), ("metabolic", 300),
                        ("twostage", 400), ("td", 400)):
        sc = load_scenario(os.path.join(SCEN, f"{name}.toy"))
        mesh = sc.build_mesh()
        save_run(f"scen_{name}", mesh, sc.material, sc.boundary, sc.initial_temperature, steps,
                 dt=sc.dt, td_mode=sc.td_mode, probes=mesh.node_sets["center"], interval=20)

    # BASELINE config 1: hex 20^3, fp64, constant props, Pennes, Gaussian source
    # lumped as Q(x_i) * v_i on one-node load sets, Dirichlet 37 on all faces,
    # dt = 0.9 * Gershgorin limit, 1000 steps.
    base = generate_cube_mesh("hex", 20, 0.1)
    vols = fedheat.node_volume_shares(base)
    d2 = ((base.nodes - 0.05) ** 2).sum(axis=1)
    q = 5.0e6 * np.exp(-d2 / (2.0 * 0.005 ** 2)) * vols
    sets = dict(base.node_sets)
    loads = []
    for i in np.nonzero(q > 0.0)[0]:
        sets[f"g{i}"] = np.array([i])
        loads.append((f"g{i}", float(q[i]), 0.0, 1.0e30))
    mesh = Mesh(nodes=base.nodes, tets=base.tets, hexes=base.hexes, node_sets=sets)
    mat1 = TissueMaterial.constant(density=1060.0, specific_heat=3600.0, conductivity=0.5,
                                   perfusion_rate=0.5e-3 * 1050.0, blood_specific_heat=3640.0,
                                   arterial_temperature=37.0, metabolic_rate=420.0)
    faces = tuple((f, 37.0) for f in ("x0", "x1", "y0", "y1", "z0", "z1"))
    probes = np.r_[base.node_sets["center"], [0, 4630, 5000, 9000]]
    save_run("cfg1", mesh, mat1, BoundarySpec(dirichlet=faces, heat_loads=tuple(loads)), 37.0, 1000,
             auto=0.9, probes=probes, interval=1, extra={"q_static": q})

    # config 2 (reference-expressible part): linear k(T), c(T) as 2-knot curves
    # on [0, 2000] C, source peak 2e7, 2000 steps, fp64.
    xs = np.array([0.0, 2000.0])
    mat2 = TissueMaterial(
        density=PropertyCurve([0.0], [1060.0]),
        specific_heat=PropertyCurve(xs, 3600.0 * (1.0 - 0.0005 * (xs - 37.0))),
        conductivity=PropertyCurve(xs, 0.5 * (1.0 + 0.0013 * (xs - 37.0))),
        perfusion_rate=0.5e-3 * 1050.0, blood_specific_heat=3640.0, arterial_temperature=37.0,
        metabolic_rate=420.0)
    loads2 = tuple((n, p * 4.0, a, b) for n, p, a, b in loads)
    save_run("cfg2", mesh, mat2, BoundarySpec(dirichlet=faces, heat_loads=loads2), 37.0, 2000,
             dt=56.342741836257446, probes=probes, interval=10, extra={"q_static": q * 4.0})


def gen_critical_dt():
    rng = np.random.default_rng(99)
    out = {}
    td = TissueMaterial(density=PropertyCurve([37.0, 65.0], [1040.0, 1000.0]),
                        specific_heat=PropertyCurve([37.0, 65.0], [3600.0, 3800.0]),
                        conductivity=PropertyCurve([37.0, 65.0], [0.53, 0.57]), perfusion_rate=26.6)
    for case in range(6):
        mesh = mixed_mesh(rng, 3, float(rng.uniform(0.02, 1.0)))
        T = rng.uniform(20.0, 60.0, mesh.n_nodes)
        eng = ExplicitEngine(mesh, td)
        for k, v in mesh_dict(mesh).items():
            out[f"c{case}_{k}"] = v
        out[f"c{case}_T"] = T
        out[f"c{case}_dt"] = np.float64(eng.critical_dt(T))
    out.update(mat_dict(td))
    np.savez_compressed(os.path.join(OUT, "critical_dt.npz"), **out)
    print("critical_dt")


def gen_instability():
    mesh = generate_cube_mesh("tet", 3, 0.01)
    mat = TissueMaterial.constant(density=1060.0, specific_heat=3700.0, conductivity=0.518)
    eng = ExplicitEngine(mesh, mat)
    dt = 10.0 * eng.critical_dt(37.0)
    T0 = 37.0 + 0.01 * np.sin(np.arange(mesh.n_nodes))
    st = eng.initial_state(T0)
    fail = None
    for _ in range(2000):
        try:
            eng.step(st, dt)
        except InstabilityError as err:
            fail = (err.step, err.node)
            break
    np.savez_compressed(os.path.join(OUT, "instability.npz"), **mesh_dict(mesh), **mat_dict(mat),
                        T0=T0, dt=np.float64(dt), fail_step=np.int64(fail[0]), fail_node=np.int64(fail[1]),
                        T_fail=st.temperatures)
    print("instability", fail)


if __name__ == "__main__":
    fedheat.kernels.warmup()
    gen_precompute()
    gen_scatter()
    gen_critical_dt()
    gen_instability()
    gen_runs()
