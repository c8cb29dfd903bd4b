"""INTEGRATION.md's operator-layer stub, dropped into the REAL reference package.

The reference package (pip-installed into baseline/_ref by
scripts/vendor_reference_suite.sh; git-ignored, it travels to the GPU box) is
copied to a temp dir, and the ctypes stub of INTEGRATION.md section 1 --
extracted verbatim from the markdown -- replaces the five numba kernel bodies
of its fedheat/kernels.py (kernels.py:76-142; the worker-control helpers stay).
The reference's own solver then runs a bundled scenario with every kernel call
going through libfedheat_b200.so, and the result must equal the reference's
golden run bit for bit.  `element_mean_nodal` (the TD refresh's kbar) is also
called directly.
"""

import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "baseline", "_ref", "fedheat")
LIB = os.path.join(ROOT, "paper_1909_05098_b200", "libfedheat_b200.so")

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {golden_dir!r})
import fedheat
from fedheat import kernels
from fedheat.material import PropertyCurve, TissueMaterial
from fedheat.mesh import Mesh
from fedheat.solver import BoundarySpec, ExplicitEngine

assert "libfedheat_b200" in repr(kernels._L), "stub not active"
for tag in ("scen_td", "scen_twostage"):
    with np.load({golden_dir!r} + f"/run_{{tag}}.npz") as z:
        d = {{k: z[k] for k in z.files}}
    sets, dirichlet, heat = {{}}, [], []
    for k, v in enumerate(np.unique(d["dir_vals"])):
        sets[f"dir{{k}}"] = d["dir_nodes"][d["dir_vals"] == v]
        dirichlet.append((f"dir{{k}}", float(v)))
    offs = d["load_offs"]
    for i in range(len(offs) - 1):
        sets[f"load{{i}}"] = d["load_nodes"][offs[i]:offs[i + 1]]
        heat.append((f"load{{i}}", float(d["load_power"][i]), float(d["load_t0"][i]), float(d["load_t1"][i])))
    mesh = Mesh(nodes=d["nodes"], tets=d["tets"], hexes=d["hexes"], node_sets=sets)
    c = lambda n: PropertyCurve(d[f"mat_{{n}}_x"], d[f"mat_{{n}}_y"])
    mat = TissueMaterial(density=c("density"), specific_heat=c("specific_heat"), conductivity=c("conductivity"),
                         perfusion_rate=float(d["mat_perfusion_rate"]),
                         blood_specific_heat=float(d["mat_blood_specific_heat"]),
                         arterial_temperature=float(d["mat_arterial_temperature"]),
                         metabolic_rate=float(d["mat_metabolic_rate"]))
    eng = ExplicitEngine(mesh, mat, BoundarySpec(dirichlet=tuple(dirichlet), heat_loads=tuple(heat)),
                         td_mode=bool(d["td_mode"]))
    res = eng.run(d["T0"], steps=int(d["steps"]), dt=float(d["dt"]), probes=d["probes"],
                  probe_interval=int(d["interval"]))
    assert np.array_equal(res.state.temperatures, d["T_final"]), tag
    assert np.array_equal(res.probe_values, d["probe_values"]), tag
    packed = eng.packed
    rng = np.random.default_rng(5)
    nodal = rng.uniform(0.4, 0.6, mesh.n_nodes)
    out = np.empty(packed.n_elements)
    kernels.element_mean_nodal(packed.conn_data, packed.conn_offs, nodal, out)
    ref = np.empty(packed.n_elements)
    for e in range(packed.n_elements):  # kernels.py:90-98: s = 0.0; s += ... in local-node order
        a, b = int(packed.conn_offs[e]), int(packed.conn_offs[e + 1])
        s = 0.0
        for p in range(a, b):
            s += float(nodal[packed.conn_data[p]])
        ref[e] = s / (b - a)
    assert np.array_equal(out, ref), "element_mean_nodal"
print("STUB-OK")
"""


def stub_source():
    with open(os.path.join(ROOT, "INTEGRATION.md")) as f:
        md = f.read()
    m = re.search(r"```python\n(# fedheat/kernels\.py.*?)```", md, re.S)
    assert m, "INTEGRATION.md has no kernels.py stub block"
    return m.group(1).replace("/path/to/paper_1909_05098_b200/libfedheat_b200.so", LIB)


@pytest.mark.skipif(not os.path.isdir(REF_PKG), reason="reference package not staged (scripts/vendor_reference_suite.sh)")
def test_integration_stub_inside_reference(tmp_path):
    pkg = tmp_path / "fedheat"
    shutil.copytree(REF_PKG, pkg)
    with open(pkg / "kernels.py") as f:
        original = f.read()
    with open(pkg / "kernels.py", "w") as f:
        f.write(original + "\n\n# ---- GPU bodies: INTEGRATION.md section 1 (replaces kernels.py:76-142) ----\n")
        f.write(stub_source())
    env = dict(os.environ, PYTHONPATH=str(tmp_path), NUMBA_CACHE_DIR=str(tmp_path / "numba_cache"))
    script = SCRIPT.format(golden_dir=os.path.join(ROOT, "tests", "golden"))
    out = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "STUB-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-4000:]
