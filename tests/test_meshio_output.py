"""Mesh ingest and run outputs vs the reference's own outputs (CPU only).

Fixtures: tests/golden/make_golden_io.py ran the reference parser
(mesh.py:153-256), VTK writer (vtkio.py:20-57) and `fedheat run`
(cli.py:95-168).  The native reader / formatter (csrc/fh_meshio.cpp) must
reproduce them byte for byte: same parsed arrays, same error class, message
and line, same file bytes.
"""

import json
import math
import os
from types import SimpleNamespace

import numpy as np
import pytest

import paper_1909_05098_b200 as fh
from paper_1909_05098_b200 import meshio, output

IO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def read(*parts) -> str:
    with open(os.path.join(IO, *parts), newline="") as f:
        return f.read()


CASES = json.loads(read("parse_cases.json"))


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_parse_matches_reference(case):
    exp = case["expect"]
    if "ok" in exp:
        mesh = meshio.parse_mesh_text(case["text"])
        assert meshio.serialize_mesh_text(mesh) == exp["ok"]
        return
    with pytest.raises(fh.FedheatError) as info:
        meshio.parse_mesh_text(case["text"])
    err = info.value
    assert type(err).__name__ == exp["error"]
    assert str(err) == exp["message"]
    assert getattr(err, "line", None) == exp["line"]


def test_parse_threads_and_file(tmp_path):
    text = read("mesh_mixed.txt")
    path = tmp_path / "m.txt"
    path.write_text(text)
    a = meshio.parse_mesh(path, threads=1)
    b = meshio.parse_mesh_text(text, threads=7)
    for x, y in ((a.nodes, b.nodes), (a.tets, b.tets), (a.hexes, b.hexes)):
        assert np.array_equal(x, y)
    assert a.node_sets.keys() == b.node_sets.keys()


def test_serialize_byte_identical(tmp_path):
    text = read("mesh_mixed.txt")
    mesh = meshio.parse_mesh_text(text)
    assert meshio.serialize_mesh_text(mesh) == text
    meshio.serialize_mesh(mesh, tmp_path / "out.txt")
    assert (tmp_path / "out.txt").read_text() == text


def test_large_parse_roundtrip_many_threads():
    """A mesh big enough for the threaded coordinate pass (> 4096 nodes)."""
    mesh = fh.jittered_cube_mesh("tet", 18, 0.1, jitter=0.2, seed=3)
    text = meshio.serialize_mesh_text(mesh)
    back = meshio.parse_mesh_text(text, threads=8)
    assert np.array_equal(back.nodes, mesh.nodes)
    assert np.array_equal(back.tets, mesh.tets)
    assert meshio.serialize_mesh_text(back) == text
    # corrupt one coordinate deep in the block: the earliest bad token wins
    lines = text.split("\n")
    lines[4001] = lines[4001].split(" ")[0] + " 1.0.0 " + lines[4001].split(" ")[2]
    lines[5001] = "bad " + lines[5001]
    with pytest.raises(fh.MeshFormatError) as info:
        meshio.parse_mesh_text("\n".join(lines), threads=8)
    assert info.value.line == 4002
    assert "coordinate of node 4000, got '1.0.0'" in str(info.value)


def test_npz_roundtrip(tmp_path):
    mesh = meshio.parse_mesh_text(read("mesh_mixed.txt"))
    meshio.save_mesh_npz(mesh, tmp_path / "m.npz")
    back = meshio.load_mesh_npz(tmp_path / "m.npz")
    assert meshio.serialize_mesh_text(back) == meshio.serialize_mesh_text(mesh)


def test_repr_formatter_special_values():
    vals = np.array([0.0, -0.0, 1.0, 1e16, 1e15, 1e-4, 1e-5, 5e-324, 1.7976931348623157e308, 0.1, 1 / 3,
                     2.0 ** -1022, 2.0 ** 60, -37.5, np.inf, -np.inf, np.nan, 123456789012345678.0])
    assert meshio.format_rows_f64(vals) == "".join(repr(float(v)) + "\n" for v in vals)
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2 ** 63, 20000, dtype=np.int64).view(np.float64)
    pw = np.ldexp(1.0, np.arange(-1074, 1024))
    for v in (bits, pw, 37.0 + rng.standard_normal(20000), rng.random(20000) * 0.3):
        assert meshio.format_rows_f64(v) == "".join(repr(float(x)) + "\n" for x in v)
    ints = rng.integers(-2 ** 63, 2 ** 63 - 1, size=(50, 8), dtype=np.int64)
    assert meshio.format_rows_i64(ints, " ", "hex8 ") == "".join(
        "hex8 " + " ".join(map(str, r)) + "\n" for r in ints)


def test_vtk_byte_identical(tmp_path):
    mesh = meshio.parse_mesh_text(read("mesh_mixed.txt"))
    with np.load(os.path.join(IO, "vtk_mixed_fields.npz")) as z:
        fields = {"temperature": z["temperature"], "k field": z["k_field"]}
    text = output.vtk_text(mesh, fields, title="mixed t=0.5 s\nsecond line")
    assert text == read("vtk_mixed.vtk")
    output.write_vtk(tmp_path / "a.vtk", mesh, fields, title="mixed t=0.5 s\nsecond line")
    assert (tmp_path / "a.vtk").read_text() == text
    with pytest.raises(fh.ConfigError):
        output.vtk_text(mesh, {"t": np.zeros(3)})


def reference_result():
    with np.load(os.path.join(IO, "conduction", "run.npz")) as z:
        d = {k: z[k] for k in z.files}
    man = json.loads(read("conduction", "manifest.json"))
    state = SimpleNamespace(temperatures=d["T_final"], time=float(d["time"]), step_index=int(d["step_index"]))
    res = SimpleNamespace(state=state, dt=float(d["dt"]), n_steps=int(d["n_steps"]),
                          dt_critical=float(d["dt_critical"]), td_mode=bool(d["td_mode"]),
                          workers=int(d["workers"]), probe_nodes=d["probe_nodes"], probe_times=d["probe_times"],
                          probe_values=d["probe_values"], timings=man["timings_s"])
    return res, man


def test_run_outputs_byte_identical(tmp_path):
    res, man = reference_result()
    mesh = fh.generate_cube_mesh("tet", 10, 0.1)
    writer = output.SnapshotWriter(tmp_path, mesh, "conduction")
    writer(res.state)
    writer.close()
    got = output.write_run_outputs(tmp_path, res, scenario_name="conduction", mesh=mesh,
                                   mesh_source=man["mesh"]["source"], version=man["fedheat_version"],
                                   snapshots=man["snapshots"])
    for name in ("probes.csv", "stats.csv", "manifest.json", "snapshot_000400.vtk"):
        assert (tmp_path / name).read_text() == read("conduction", name), name
    assert got["final_field_sha256"] == man["final_field_sha256"]
    assert output.stats_summary(res.state.temperatures) == man["final_field_stats"]
    assert math.isfinite(got["final_field_stats"]["rms"])
    with pytest.raises(fh.ConfigError):
        output.stats_summary(np.empty(0))
