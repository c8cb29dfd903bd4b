"""Run outputs in the reference's wire formats.

What `fedheat run` writes (/root/reference/pkg/src/fedheat/cli.py:95-168),
byte for byte, for a `RunResult` of this engine:

* `probes.csv`  -- cli.py:81-86: ``time_s,node_<id>...`` then repr() rows;
* `stats.csv`   -- cli.py:150-154 with oracle.py:274-287 `stats_summary`
  (numpy linear-interpolation quartiles and the RMS);
* `snapshot_<step:06d>.vtk` -- vtkio.py:20-57 legacy ASCII VTK 2.0;
* `manifest.json` -- cli.py:137-161, including `final_field_sha256`, the
  SHA-256 of the float64 field bytes (the reference's determinism check).

Numbers are rendered by the native formatter (`fh_format_f64`, Python repr
semantics, all host threads).  `SnapshotWriter` renders the mesh part of the
VTK file once and formats each snapshot on a background thread (the native
call releases the GIL), so the GPU keeps stepping while the previous
snapshot is written.
"""

from __future__ import annotations

import hashlib
import json
import math
import threading
from concurrent.futures import Future, ThreadPoolExecutor
from pathlib import Path

import numpy as np

from .errors import ConfigError
from .mesh import Mesh
from .meshio import format_rows_f64, format_rows_i64

_CELL_TYPE_TET = 10
_CELL_TYPE_HEX = 12
STATS_KEYS = ("min", "q1", "median", "q3", "max", "rms")


# ------------------------------------------------------------------ VTK --
def _vtk_title(title: str) -> str:
    return title.splitlines()[0][:255] if title else "fedheat snapshot"


def vtk_mesh_text(mesh: Mesh, title: str = "fedheat snapshot") -> str:
    """Everything of vtkio.py:20-41 before POINT_DATA (header, points, cells)."""
    n_cells = mesh.n_elements
    total = mesh.tets.size + mesh.tets.shape[0] + mesh.hexes.size + mesh.hexes.shape[0]
    parts = [
        "# vtk DataFile Version 2.0\n", _vtk_title(title) + "\n", "ASCII\n", "DATASET UNSTRUCTURED_GRID\n",
        f"POINTS {mesh.n_nodes} double\n", format_rows_f64(mesh.nodes, " "),
        f"CELLS {n_cells} {total}\n",
    ]
    if mesh.tets.size:
        parts.append(format_rows_i64(mesh.tets, " ", "4 "))
    if mesh.hexes.size:
        parts.append(format_rows_i64(mesh.hexes, " ", "8 "))
    parts.append(f"CELL_TYPES {n_cells}\n")
    parts.append(f"{_CELL_TYPE_TET}\n" * mesh.tets.shape[0])
    parts.append(f"{_CELL_TYPE_HEX}\n" * mesh.hexes.shape[0])
    return "".join(parts)


def vtk_point_data_text(mesh: Mesh, point_data: dict) -> str:
    """The POINT_DATA block of vtkio.py:43-52."""
    if not point_data:
        return ""
    parts = [f"POINT_DATA {mesh.n_nodes}\n"]
    for name, values in point_data.items():
        values = np.asarray(values, dtype=np.float64)
        if values.shape != (mesh.n_nodes,):
            raise ConfigError(f"field {name!r} has shape {values.shape}, expected ({mesh.n_nodes},)")
        safe = name.replace(" ", "_")
        parts.append(f"SCALARS {safe} double 1\nLOOKUP_TABLE default\n")
        parts.append(format_rows_f64(values))
    return "".join(parts)


def _split_title_line(mesh_text: str, title: str) -> str:
    head, rest = mesh_text.split("\n", 2)[0], mesh_text.split("\n", 2)[2]
    return f"{head}\n{_vtk_title(title)}\n{rest}"


def vtk_text(mesh: Mesh, point_data: dict, title: str = "fedheat snapshot") -> str:
    """vtkio.py:20-52 vtk_text: byte-identical legacy ASCII VTK."""
    return vtk_mesh_text(mesh, title) + vtk_point_data_text(mesh, point_data)


def write_vtk(path, mesh: Mesh, point_data: dict, title: str = "fedheat snapshot") -> None:
    """vtkio.py:55-57 write_vtk."""
    Path(path).write_text(vtk_text(mesh, point_data, title))


class SnapshotWriter:
    """`on_snapshot` callback writing cli.py:116-124's snapshot files.

    The mesh text (points, cells) is rendered once; each snapshot formats only
    its temperature field, on a worker thread when `background` is true.  Call
    `close()` (or use as a context manager) to wait for pending writes.
    """

    def __init__(self, out_dir, mesh: Mesh, scenario_name: str, background: bool = True):
        self.out_dir = Path(out_dir)
        self.out_dir.mkdir(parents=True, exist_ok=True)
        self.mesh = mesh
        self.name = scenario_name
        self.names: list[str] = []
        self._mesh_text = vtk_mesh_text(mesh, "x")
        self._pool = ThreadPoolExecutor(max_workers=1) if background else None
        self._pending: list[Future] = []
        self._lock = threading.Lock()

    def _write(self, path: Path, title: str, T: np.ndarray) -> None:
        body = _split_title_line(self._mesh_text, title) + vtk_point_data_text(self.mesh, {"temperature": T})
        path.write_text(body)

    def __call__(self, state) -> None:
        name = f"snapshot_{state.step_index:06d}.vtk"
        title = f"{self.name} t={state.time!r} s"
        T = np.array(state.temperatures, dtype=np.float64, copy=True)
        self.names.append(name)
        if self._pool is None:
            self._write(self.out_dir / name, title, T)
        else:
            with self._lock:
                self._pending.append(self._pool.submit(self._write, self.out_dir / name, title, T))

    def close(self) -> None:
        if self._pool is not None:
            for f in self._pending:
                f.result()
            self._pending.clear()
            self._pool.shutdown(wait=True)
            self._pool = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ------------------------------------------------------------ CSV / stats --
def stats_summary(values) -> dict:
    """oracle.py:274-287: min / linear-interpolation quartiles / max and the RMS."""
    vals = np.asarray(values, dtype=np.float64)
    if vals.size == 0:
        raise ConfigError("cannot summarize an empty field")
    q0, q1, q2, q3, q4 = np.quantile(vals, [0.0, 0.25, 0.5, 0.75, 1.0])
    return {"min": float(q0), "q1": float(q1), "median": float(q2), "q3": float(q3), "max": float(q4),
            "rms": float(math.sqrt(float(np.mean(vals * vals))))}


def format_stats(stats: dict) -> str:
    """cli.py:89-92 console table."""
    width = max(len(k) for k in STATS_KEYS)
    return "\n".join(f"  {k.rjust(width)}: {stats[k]:.6f}" for k in STATS_KEYS)


def stats_csv_text(stats: dict) -> str:
    """cli.py:150-154."""
    return "min,q1,median,q3,max,rms\n" + ",".join(repr(stats[k]) for k in STATS_KEYS) + "\n"


def probes_csv_text(result) -> str:
    """cli.py:81-86 _write_probes_csv."""
    header = "time_s," + ",".join(f"node_{int(n)}" for n in result.probe_nodes) + "\n"
    table = np.column_stack([np.asarray(result.probe_times, dtype=np.float64),
                             np.asarray(result.probe_values, dtype=np.float64).reshape(len(result.probe_times), -1)])
    return header + format_rows_f64(table, ",")


def field_sha256(temperatures) -> str:
    """cli.py:146-148: SHA-256 of the float64 field bytes."""
    return hashlib.sha256(np.ascontiguousarray(temperatures, dtype=np.float64).tobytes()).hexdigest()


def run_manifest(result, *, scenario_name: str, mesh: Mesh, mesh_source: str, version: str,
                 stats: dict | None = None, snapshots=()) -> dict:
    """cli.py:137-161 manifest dict."""
    stats = stats_summary(result.state.temperatures) if stats is None else stats
    return {
        "fedheat_version": version,
        "scenario": scenario_name,
        "mesh": {"nodes": mesh.n_nodes, "elements": mesh.n_elements, "source": mesh_source},
        "steps": result.n_steps,
        "dt_s": result.dt,
        "dt_critical_s": result.dt_critical,
        "simulated_time_s": result.state.time,
        "td_mode": result.td_mode,
        "workers": result.workers,
        "timings_s": result.timings,
        "final_field_sha256": field_sha256(result.state.temperatures),
        "final_field_stats": stats,
        "probe_nodes": [int(n) for n in result.probe_nodes],
        "snapshots": list(snapshots),
    }


def write_run_outputs(out_dir, result, *, scenario_name: str, mesh: Mesh, mesh_source: str, version: str,
                      snapshots=()) -> dict:
    """The files cli.py:134-161 writes after a run: probes.csv (when there are
    probes), stats.csv and manifest.json.  Returns the manifest."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    stats = stats_summary(result.state.temperatures)
    if np.asarray(result.probe_nodes).size:
        (out / "probes.csv").write_text(probes_csv_text(result))
    (out / "stats.csv").write_text(stats_csv_text(stats))
    manifest = run_manifest(result, scenario_name=scenario_name, mesh=mesh, mesh_source=mesh_source,
                            version=version, stats=stats, snapshots=snapshots)
    (out / "manifest.json").write_text(json.dumps(manifest, indent=2, sort_keys=True) + "\n")
    return manifest
