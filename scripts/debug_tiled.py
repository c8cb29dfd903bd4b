"""Diagnose TILED vs EXACT differences on small meshes (GPU)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1909_05098_b200 as fh

def problem(td, loads, kind="hex", div=8):
    mesh = fh.generate_cube_mesh(kind, div, 0.1)
    if td:
        mat = fh.TissueMaterial(density=fh.make_constant(1060.0), specific_heat=fh.linear_law(3600.0, -0.0005, 37.0),
                                conductivity=fh.linear_law(0.5, 0.0013, 37.0), perfusion_rate=0.525,
                                blood_specific_heat=3640.0, metabolic_rate=420.0)
    else:
        mat = fh.TissueMaterial.constant(density=1060.0, specific_heat=3600.0, conductivity=0.5, perfusion_rate=0.525,
                                         blood_specific_heat=3640.0, metabolic_rate=420.0)
    faces = tuple((f, 37.0) for f in ("x0", "x1", "y0", "y1", "z0", "z1"))
    hl = (("center", 20.0, 0.0, 1.0e9),) if loads else ()
    return mesh, mat, fh.BoundarySpec(dirichlet=faces, heat_loads=hl)

for kind in ("hex", "tet"):
  for td in (False, True):
    for loads in (False, True):
        mesh, mat, bnd = problem(td, loads, kind)
        ex = fh.ExplicitEngine(mesh, mat, bnd)
        r = ex.run(37.0, steps=50, auto_dt_safety=0.9)
        T0 = mesh.nodes[:, 0] * 100 + 30.0
        for pn in (64, 256, 100000):
            for prec in (64, 32):
                t = fh.ExplicitEngine(mesh, mat, bnd, assembly="tiled", precision=prec, part_nodes=pn)
                rt = t.run(37.0, steps=50, dt=r.dt)
                rel = np.abs(rt.state.temperatures - r.state.temperatures).max() / np.abs(r.state.temperatures).max()
                # one step from a non-uniform field
                s1 = ex.initial_state(T0); ex.step(s1, r.dt)
                s2 = t.initial_state(T0); t.step(s2, r.dt)
                rel1 = np.abs(s1.temperatures - s2.temperatures).max() / np.abs(s1.temperatures).max()
                print(f"{kind} td={td} loads={loads} part_nodes={pn} prec={prec} layout={t.layout()['n_parts']} rel50={rel:.2e} rel1={rel1:.2e}", flush=True)
