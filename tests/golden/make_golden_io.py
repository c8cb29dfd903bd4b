"""Generate the I/O golden fixtures by running the REFERENCE package itself.

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden_io.py

Writes tests/golden/io/:
  parse_cases.json    mesh texts (valid and malformed) with the reference's
                      outcome: the re-serialized mesh (mesh.py:241-253) or the
                      exception class, message and line (mesh.py:153-236)
  mesh_mixed.txt      serialize_mesh_text of a jittered mixed tet/hex mesh
  vtk_mixed.vtk       vtkio.vtk_text of that mesh with two point fields
  conduction/         `fedheat run` (cli.py:95-168) of the bundled conduction
                      scenario, 400 steps, a snapshot every 200 steps:
                      probes.csv, stats.csv, manifest.json, snapshot_*.vtk,
                      plus run.npz with the RunResult arrays the files came from
"""

from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")

from fedheat import cli, vtkio  # noqa: E402
from fedheat.errors import FedheatError  # noqa: E402
from fedheat.mesh import Mesh, parse_mesh_text, serialize_mesh_text  # noqa: E402
from fedheat.meshgen import generate_cube_mesh  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")
SCEN = os.path.join(REF, "fedheat", "scenarios")


def mixed_mesh() -> Mesh:
    rng = np.random.default_rng(77)
    tet = generate_cube_mesh("tet", 3, 0.01)
    nodes = tet.nodes.copy()
    interior = np.all((nodes > 1e-9) & (nodes < 0.01 - 1e-9), axis=1)
    nodes[interior] += rng.uniform(-0.0006, 0.0006, size=(int(interior.sum()), 3))
    hexm = generate_cube_mesh("hex", 3, 0.01)
    # second block shifted along x: a hex cube glued next to the tet cube
    hn = hexm.nodes + np.array([0.02, 0.0, 0.0])
    n0 = nodes.shape[0]
    all_nodes = np.vstack([nodes, hn * np.array([1.0, 1.0, 1.0]) + 1e-7 * rng.standard_normal(hn.shape)])
    sets = {"z0": tet.node_sets["z0"], "center": tet.node_sets["center"],
            "hex.x1": hexm.node_sets["x1"] + n0, "empty_set": np.empty(0, np.int64)}
    return Mesh(nodes=all_nodes, tets=tet.tets, hexes=hexm.hexes + n0, node_sets=sets)


def parse_cases(mixed_text: str) -> list[tuple[str, str]]:
    small = serialize_mesh_text(generate_cube_mesh("tet", 1, 1.0))
    good = [
        ("mixed", mixed_text),
        ("cube_tet1", small),
        ("comments_crlf_tabs", "# header comment\r\nnodes 4 # count\r\n0 0 0\t1 0 0\r\n0 1 0   0 0 1#x\r\n"
                               "elements\t1\r\ntet4 0 1 2 3\r\nnodeset a_b.c-d 2\r\n3 1\r\n"),
        ("python_numbers", "nodes 4\n+0.0 -0.0 0e0\n1_0.5 .5 5.\n0 1E+1 0\n0 0 1_000\nelements 1\ntet4 0 1 2 3\n"
                           "nodeset s 1\n+3\n"),
        ("unicode_ws", "nodes 4\n0 0 0\n1 0 0 0 1 0\n0 0 1\nelements 1 tet4 0 1 2 3\n"
                       "# café comment\n"),
        ("form_feed_lines", "nodes 4\f0 0 0\v1 0 0\x1c0 1 0\x1d0 0 1\x1eelements 1\n\x1ftet4 0 1 2 3\n"),
        ("cr_only", "nodes 4\r0 0 0\r1 0 0\r0 1 0\r0 0 1\relements 1\rtet4 0 1 2 3\r"),
        ("hex_unit", "nodes 8\n0 0 0\n1 0 0\n1 1 0\n0 1 0\n0 0 1\n1 0 1\n1 1 1\n0 1 1\nelements 1\n"
                     "hex8 0 1 2 3 4 5 6 7\n"),
        ("interleaved", "nodes 8\n0 0 0\n1 0 0\n1 1 0\n0 1 0\n0 0 1\n1 0 1\n1 1 1\n0 1 1\nelements 2\n"
                        "hex8 0 1 2 3 4 5 6 7\ntet4 0 1 3 4\n"),
    ]
    bad = [
        ("empty", ""),
        ("unicode_line_count", "nodes 1\u2028\x850 0\u3000q\n"),
        ("nonascii_token", "nodes 1\n0 0 \u00e9\n"),
        ("only_comment", "# nothing\n\n"),
        ("wrong_kw", "points 4\n"),
        ("bad_count", "nodes four\n"),
        ("zero_nodes", "nodes 0\nelements 1\n"),
        ("neg_nodes", "\n\nnodes -3\n"),
        ("short_coords", "nodes 2\n0 0 0\n1 1\n"),
        ("bad_coord", "nodes 2\n0 0 0\n1 x 1\nelements 1\n"),
        ("bad_coord_late", "nodes 3\n0 0 0\n1 1 1\n\n# c\n2 2 0x10\n"),
        ("hex_float", "nodes 1\n0x1p3 0 0\n"),
        ("underscore_bad", "nodes 1\n1__0 0 0\n"),
        ("trailing_underscore", "nodes 1\n10_ 0 0\n"),
        ("missing_elements", "nodes 1\n0 0 0\nelem 1\n"),
        ("elem_count_float", "nodes 1\n0 0 0\nelements 1.0\n"),
        ("elem_zero", "nodes 1\n0 0 0\nelements 0\n"),
        ("bad_kind", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntri3 0 1 2\n"),
        ("bad_conn", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2.0 3\n"),
        ("eof_conn", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2\n"),
        ("eof_kind", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 2\ntet4 0 1 2 3\n"),
        ("junk_after", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2 3\nfoo\n"),
        ("bad_set_name", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2 3\nnodeset 9a 1\n0\n"),
        ("quote_token", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2 3\nit's\n"),
        ("dup_set", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2 3\nnodeset a 1\n0\n"
                    "nodeset a 1\n1\n"),
        ("set_neg_count", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2 3\nnodeset a -1\n"),
        ("set_repeat", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2 3\nnodeset a 3\n0 1\n\n0\n"),
        ("set_range", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2 3\nnodeset a 2\n0 4\n"),
        ("set_eof", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2 3\nnodeset a 3\n0 1\n"),
        ("set_no_name", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2 3\nnodeset\n"),
        ("conn_range", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2 4\n"),
        ("inverted_tet", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 2 1 3\n"),
        ("nan_coord", "nodes 4\n0 0 0\n1 0 0\n0 nan 0\n0 0 1\nelements 1\ntet4 0 1 2 3\n"),
        ("inf_coord", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 -Infinity\nelements 1\ntet4 0 1 2 3\n"),
        ("repeat_node", "nodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 1 3\n"),
        ("comment_glued", "nodes 4#c\n0 0 0#c\n1 0 0\n0 1 0\n0 0 1\nelements 1\ntet4 0 1 2 3x\n"),
    ]
    return good + bad


def outcome(text: str) -> dict:
    try:
        mesh = parse_mesh_text(text)
    except FedheatError as err:
        return {"error": type(err).__name__, "message": str(err), "line": getattr(err, "line", None)}
    return {"ok": serialize_mesh_text(mesh)}


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    mixed = mixed_mesh()
    mixed_text = serialize_mesh_text(mixed)
    with open(os.path.join(OUT, "mesh_mixed.txt"), "w") as fh:
        fh.write(mixed_text)
    cases = [{"name": n, "text": t, "expect": outcome(t)} for n, t in parse_cases(mixed_text)]
    with open(os.path.join(OUT, "parse_cases.json"), "w") as fh:
        json.dump(cases, fh, indent=1, ensure_ascii=True)
    rng = np.random.default_rng(5)
    fields = {"temperature": 37.0 + rng.standard_normal(mixed.n_nodes),
              "k field": np.r_[0.0, -0.0, 1e-7, 1e17, rng.random(mixed.n_nodes - 4) * 1e-3]}
    with open(os.path.join(OUT, "vtk_mixed.vtk"), "w") as fh:
        fh.write(vtkio.vtk_text(mixed, fields, title="mixed t=0.5 s\nsecond line"))
    np.savez_compressed(os.path.join(OUT, "vtk_mixed_fields.npz"), temperature=fields["temperature"],
                        k_field=fields["k field"])

    # `fedheat run` of the conduction scenario with snapshots
    run_dir = os.path.join(OUT, "conduction")
    shutil.rmtree(run_dir, ignore_errors=True)
    with tempfile.TemporaryDirectory() as tmp:
        src = open(os.path.join(SCEN, "conduction.toy")).read()
        src = src.replace("probe_interval = 20", "probe_interval = 20\nsnapshot_interval = 200")
        toy = os.path.join(tmp, "conduction.toy")
        with open(toy, "w") as fh:
            fh.write(src)
        captured = {}
        orig_run = cli.ExplicitEngine.run

        def spy(self, *a, **k):
            res = orig_run(self, *a, **k)
            captured["res"] = res
            return res

        cli.ExplicitEngine.run = spy
        try:
            rc = cli.main(["run", toy, "--steps", "400", "--output", run_dir, "--workers", "1"])
        finally:
            cli.ExplicitEngine.run = orig_run
        assert rc == 0, rc
    res = captured["res"]
    np.savez_compressed(os.path.join(run_dir, "run.npz"), T_final=res.state.temperatures,
                        probe_nodes=res.probe_nodes, probe_times=res.probe_times, probe_values=res.probe_values,
                        dt=np.float64(res.dt), dt_critical=np.float64(res.dt_critical),
                        time=np.float64(res.state.time), step_index=np.int64(res.state.step_index),
                        n_steps=np.int64(res.n_steps), td_mode=np.int64(res.td_mode), workers=np.int64(res.workers))
    print("io fixtures:", sorted(os.listdir(OUT)), sorted(os.listdir(run_dir)))


if __name__ == "__main__":
    main()
