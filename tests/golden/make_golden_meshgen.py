"""Reference fixtures for generate_cube_mesh (meshgen.py:59-116): run the
REFERENCE generator here and store its arrays (node coordinates, elements,
every node set) for tests/test_meshgen_golden.py.

    python tests/golden/make_golden_meshgen.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from fedheat.meshgen import generate_cube_mesh  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CASES = [("hex", 1, 1.0), ("hex", 2, 0.1), ("hex", 5, 0.07), ("hex", 9, 0.1), ("tet", 1, 1.0), ("tet", 2, 0.1),
         ("tet", 5, 0.03), ("tet", 8, 0.1)]

if __name__ == "__main__":
    for kind, div, size in CASES:
        m = generate_cube_mesh(kind, div, size)
        d = {"nodes": m.nodes, "tets": m.tets, "hexes": m.hexes, "kind": kind, "div": div, "size": size}
        for name, ids in m.node_sets.items():
            d[f"set_{name}"] = np.asarray(ids)
        path = os.path.join(OUT, f"meshgen_{kind}{div}.npz")
        np.savez_compressed(path, **d)
        print(path, m.nodes.shape, m.tets.shape, m.hexes.shape, sorted(m.node_sets))
