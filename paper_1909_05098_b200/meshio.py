"""Mesh ingest and text rendering at scale.

* `parse_mesh_text` / `parse_mesh`: the reference's mesh file grammar
  (/root/reference/pkg/src/fedheat/mesh.py:153-239), parsed by the native
  C++ reader `fh_mesh_parse` (csrc/fh_meshio.cpp): same tokens, same error
  messages and line numbers, the coordinate block converted by all host
  threads.  The reference's Python token generator needs minutes for a
  25 M-element file; the native reader takes seconds.
* `serialize_mesh_text` / `serialize_mesh`: mesh.py:241-256, byte-identical
  output (Python repr of every coordinate, str of every index) rendered by
  `fh_format_f64` / `fh_format_i64`.
* `save_mesh_npz` / `load_mesh_npz`: a binary container (numpy .npz, no
  pickling) for meshes too large for text; not in the reference.

`format_rows_f64` / `format_rows_i64` are the shared text renderers that the
VTK, probes.csv and stats writers in `output.py` use.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import _native as N
from .errors import FH_ERR_FORMAT, MeshFormatError
from .mesh import Mesh

_ROWS_PER_BLOCK = 1 << 20


def _render(fn, arr, ptr_type, sep: str, prefix: str | None, threads: int, max_len: int) -> str:
    rows, cols = arr.shape
    if rows == 0:
        return ""
    pre = None if not prefix else prefix.encode()
    row_max = (len(pre) if pre else 0) + cols * (max_len + 1) + 1
    pieces = []
    for lo in range(0, rows, _ROWS_PER_BLOCK):
        blk = np.ascontiguousarray(arr[lo:lo + _ROWS_PER_BLOCK])
        cap = blk.shape[0] * row_max
        buf = np.empty(cap, dtype=np.uint8)
        used = C.c_int64(0)
        N.check(fn(blk.ctypes.data_as(ptr_type), blk.shape[0], cols, sep.encode(), pre, threads,
                   buf.ctypes.data_as(C.c_char_p), cap, C.byref(used)))
        pieces.append(buf[:used.value].tobytes().decode("ascii"))
    return "".join(pieces)


def format_rows_f64(values, sep: str = " ", prefix: str | None = None, threads: int = 0) -> str:
    """Rows of Python repr(float) values joined by `sep`, each row ending in newline."""
    arr = np.asarray(values, dtype=np.float64)
    arr = arr.reshape(arr.shape[0], -1) if arr.ndim != 1 else arr.reshape(-1, 1)
    return _render(N.lib().fh_format_f64, arr, N.f64p, sep, prefix, threads, 25)


def format_rows_i64(values, sep: str = " ", prefix: str | None = None, threads: int = 0) -> str:
    """Rows of str(int) values joined by `sep`, each row ending in newline."""
    arr = np.asarray(values, dtype=np.int64)
    arr = arr.reshape(arr.shape[0], -1) if arr.ndim != 1 else arr.reshape(-1, 1)
    return _render(N.lib().fh_format_i64, arr, N.i64p, sep, prefix, threads, 20)


def parse_mesh_bytes(data: bytes, threads: int = 0) -> Mesh:
    """Parse UTF-8 mesh text (mesh.py:192-236) with the native reader."""
    L = N.lib()
    h = C.c_void_p()
    line = C.c_int64(-1)
    status = L.fh_mesh_parse(data, len(data), threads, C.byref(h), C.byref(line))
    if status == FH_ERR_FORMAT:
        raise MeshFormatError(L.fh_last_error().decode("utf-8", "replace"),
                              line=None if line.value < 0 else int(line.value))
    N.check(status)
    try:
        nv, nt, nh = C.c_int64(), C.c_int64(), C.c_int64()
        ns = C.c_int32()
        N.check(L.fh_mesh_text_info(h, C.byref(nv), C.byref(nt), C.byref(nh), C.byref(ns)))
        nodes = np.empty((nv.value, 3), dtype=np.float64)
        tets = np.empty((nt.value, 4), dtype=np.int64)
        hexes = np.empty((nh.value, 8), dtype=np.int64)
        N.check(L.fh_mesh_text_arrays(h, N.ptr(nodes), N.ptr(tets, N.i64p), N.ptr(hexes, N.i64p)))
        sets = {}
        for i in range(ns.value):
            cnt = C.c_int64()
            name = C.create_string_buffer(4096)
            N.check(L.fh_mesh_text_set(h, i, name, 4096, None, C.byref(cnt)))
            ids = np.empty(cnt.value, dtype=np.int64)
            N.check(L.fh_mesh_text_set(h, i, name, 4096, N.ptr(ids, N.i64p), C.byref(cnt)))
            sets[name.value.decode("utf-8")] = ids
    finally:
        L.fh_mesh_text_destroy(h)
    return Mesh(nodes=nodes, tets=tets, hexes=hexes, node_sets=sets)


def parse_mesh_text(text: str, threads: int = 0) -> Mesh:
    """mesh.py:192 parse_mesh_text(text) -> Mesh."""
    return parse_mesh_bytes(text.encode("utf-8", "surrogatepass"), threads)


def parse_mesh(path, threads: int = 0) -> Mesh:
    """mesh.py:238 parse_mesh(path) -> Mesh (the file is read as bytes)."""
    return parse_mesh_bytes(Path(path).read_bytes(), threads)


def serialize_mesh_text(mesh: Mesh, threads: int = 0) -> str:
    """mesh.py:241-253: the file format back, coordinates at full precision."""
    out = [f"nodes {mesh.n_nodes}\n", format_rows_f64(mesh.nodes, " ", None, threads),
           f"elements {mesh.n_elements}\n"]
    if mesh.tets.size:
        out.append(format_rows_i64(mesh.tets, " ", "tet4 ", threads))
    if mesh.hexes.size:
        out.append(format_rows_i64(mesh.hexes, " ", "hex8 ", threads))
    for name in sorted(mesh.node_sets):
        ids = mesh.node_sets[name]
        out.append(f"nodeset {name} {ids.size}\n")
        full = ids.size // 8 * 8
        if full:
            out.append(format_rows_i64(ids[:full].reshape(-1, 8), " ", None, threads))
        if ids.size > full:
            out.append(format_rows_i64(ids[full:].reshape(1, -1), " ", None, threads))
    return "".join(out)


def serialize_mesh(mesh: Mesh, path, threads: int = 0) -> None:
    """mesh.py:255-256."""
    Path(path).write_text(serialize_mesh_text(mesh, threads))


def save_mesh_npz(mesh: Mesh, path) -> None:
    """Binary mesh container: nodes, tets, hexes and one `set:<name>` array per node set."""
    arrays = {"nodes": mesh.nodes, "tets": mesh.tets, "hexes": mesh.hexes}
    for name, ids in mesh.node_sets.items():
        arrays[f"set:{name}"] = ids
    with open(path, "wb") as fh:
        np.savez(fh, **arrays)


def load_mesh_npz(path) -> Mesh:
    """Inverse of `save_mesh_npz`; the mesh is validated like any other Mesh."""
    with np.load(path, allow_pickle=False) as z:
        for key in ("nodes", "tets", "hexes"):
            if key not in z.files:
                raise MeshFormatError(f"{path}: missing array {key!r}")
        sets = {k[4:]: z[k] for k in z.files if k.startswith("set:")}
        return Mesh(nodes=z["nodes"], tets=z["tets"], hexes=z["hexes"], node_sets=sets)
