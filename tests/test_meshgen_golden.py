"""generate_cube_mesh (north_star: connectivity bookkeeping bit-exact) against
fixtures produced by the reference's own generator
(tests/golden/make_golden_meshgen.py, reference meshgen.py:59-116): node
coordinates, element connectivity and every node set, bit for bit."""
import glob
import os

import numpy as np
import pytest

import paper_1909_05098_b200 as fh

GOLD = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "meshgen_*.npz")))


@pytest.mark.parametrize("path", GOLD, ids=[os.path.basename(p)[8:-4] for p in GOLD])
def test_generate_cube_mesh_bitwise(path):
    d = np.load(path)
    m = fh.generate_cube_mesh(str(d["kind"]), int(d["div"]), float(d["size"]))
    assert m.nodes.dtype == d["nodes"].dtype and np.array_equal(m.nodes, d["nodes"])
    assert np.array_equal(m.tets.reshape(-1, 4), d["tets"].reshape(-1, 4))
    assert np.array_equal(m.hexes.reshape(-1, 8), d["hexes"].reshape(-1, 8))
    sets = {k[4:] for k in d.files if k.startswith("set_")}
    assert sets == set(m.node_sets)
    for name in sets:
        assert np.array_equal(np.asarray(m.node_sets[name]), d[f"set_{name}"]), name


def test_fixture_count():
    assert len(GOLD) == 8
