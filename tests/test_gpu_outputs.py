"""`fedheat run` outputs from the GPU engine, byte for byte vs the reference.

The reference CLI ran the bundled conduction scenario for 400 steps with a
snapshot every 200 steps (tests/golden/make_golden_io.py).  The EXACT-mode
engine is bitwise identical to the reference, so probes.csv, stats.csv, every
snapshot VTK and the manifest (final_field_sha256 included; timings and the
worker count aside) must be byte-identical.
"""

import json
import os

import numpy as np
import pytest

from golden_io import load

pytestmark = pytest.mark.gpu

fh = pytest.importorskip("paper_1909_05098_b200")
from paper_1909_05098_b200 import output  # noqa: E402
from test_gpu_parity import golden_problem  # noqa: E402
from golden_io import material  # noqa: E402

IO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io", "conduction")


def test_conduction_run_outputs_byte_identical(tmp_path):
    d = load("run_scen_conduction.npz")
    man = json.loads(open(os.path.join(IO, "manifest.json")).read())
    mesh, bnd = golden_problem(d)
    eng = fh.ExplicitEngine(mesh, material(d), bnd)
    with output.SnapshotWriter(tmp_path, mesh, "conduction") as writer:
        res = eng.run(37.0, steps=400, dt=0.005, probes=man["probe_nodes"], probe_interval=20,
                      snapshot_interval=200, on_snapshot=writer)
    assert writer.names == man["snapshots"]
    got = output.write_run_outputs(tmp_path, res, scenario_name="conduction", mesh=mesh,
                                   mesh_source=man["mesh"]["source"], version=man["fedheat_version"],
                                   snapshots=writer.names)
    for name in ["probes.csv", "stats.csv", *man["snapshots"]]:
        want = open(os.path.join(IO, name)).read()
        assert (tmp_path / name).read_text() == want, name
    for key in ("timings_s", "workers"):
        got.pop(key)
        man.pop(key)
    assert got == man
    assert np.array_equal(res.state.temperatures, load("run_scen_conduction.npz")["T_final"])
