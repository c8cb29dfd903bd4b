"""Run the reference's OWN test files against this repo's GPU facade.

`scripts/vendor_reference_suite.sh` (run where /root/reference exists) copies
/root/reference/pkg/tests/{test_solver,test_acceptance,test_element,
test_material,test_mesh,test_meshgen,test_precompute,test_vtkio,oracles}.py
unmodified into tests/reference_suite/vendored/ and pip-installs the reference
package into baseline/_ref/.  Both are git-ignored (reference sources are not
committed) and travel to the GPU box with the gpurun snapshot.

This conftest makes `import fedheat...` in those files resolve to:

  fedheat.solver / kernels / element / material / mesh / meshgen /
  precompute / errors / vtkio        -> paper_1909_05098_b200 (the product:
                                        every step runs on the GPU, EXACT mode)
  fedheat.oracle / cli / bench /      -> the installed reference modules
  scenario                              (test infrastructure: the implicit
                                        scipy oracle, the CLI front end); their
                                        own `from .solver import ...` resolve to
                                        the facade too, so the CLI drives the
                                        GPU engine

Every collected item is marked `gpu`.  Items that measure the reference's
CPU worker pool, or need the reference's own CPU internals, are skipped with
the reason listed in SKIPS.
"""

from __future__ import annotations

import importlib
import importlib.util
import os
import sys
import types

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
VENDORED = os.path.join(HERE, "vendored")
REF_PKG = os.path.join(ROOT, "baseline", "_ref", "fedheat")

# reason per test id (substring match on the node id)
SKIPS = {
    "test_acceptance.py::test_08a_parallel_speedup":
        "times the reference's numba worker pool (CPU threads); the GPU engine accepts and ignores `workers`",
    "test_acceptance.py::test_08b_constant_properties_step_faster":
        "CPU wall-clock comparison of the reference's TI vs TD kernels; GPU step times are in bench.py",
    "test_acceptance.py::test_08c_per_step_time_scales_linearly":
        "CPU per-node timing regression of the reference's kernels; GPU scaling is in bench.py",
}


def _install_aliases() -> bool:
    if "fedheat" in sys.modules and getattr(sys.modules["fedheat"], "__fh_alias__", False):
        return True
    if not os.path.isdir(REF_PKG):
        return False
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import paper_1909_05098_b200 as fh
    from paper_1909_05098_b200 import (element, errors, kernels, material, mesh, meshgen, meshio, precompute,
                                       solver, vtkio)

    # facade modules under the reference's module names (registered first, so
    # the reference's own `from .solver import ...` statements bind to them)
    mesh_mod = types.ModuleType("fedheat.mesh")  # Mesh + the text parser / writer (meshio.py)
    mesh_mod.__dict__.update({k: v for k, v in vars(mesh).items() if not k.startswith("__")})
    for name in ("parse_mesh_text", "parse_mesh", "serialize_mesh_text", "serialize_mesh"):
        setattr(mesh_mod, name, getattr(meshio, name))
    # the reference's private lattice tables (tests/oracles.py random_mixed_mesh
    # imports them); same values under this repo's public names
    gen_mod = types.ModuleType("fedheat.meshgen")
    gen_mod.__dict__.update({k: v for k, v in vars(meshgen).items() if not k.startswith("__")})
    gen_mod._TET_PATTERNS = list(meshgen.KUHN_PATTERNS)
    gen_mod._HEX_OFFSETS = meshgen.HEX_CORNER_OFFSETS
    aliases = {"solver": solver, "kernels": kernels, "element": element, "material": material, "mesh": mesh_mod,
               "meshgen": gen_mod, "precompute": precompute, "errors": errors, "vtkio": vtkio}
    for name, mod in aliases.items():
        sys.modules[f"fedheat.{name}"] = mod
    # the package itself is the reference's __init__ (a real file package, so
    # importlib.resources finds the bundled scenarios); everything it does not
    # find in sys.modules (scenario, and later oracle / cli / bench) loads from
    # the installed reference as test infrastructure
    spec = importlib.util.spec_from_file_location("fedheat", os.path.join(REF_PKG, "__init__.py"),
                                                  submodule_search_locations=[REF_PKG])
    pkg = importlib.util.module_from_spec(spec)
    sys.modules["fedheat"] = pkg
    spec.loader.exec_module(pkg)
    for name, mod in aliases.items():
        setattr(pkg, name, mod)
    for name in ("oracle", "scenario", "cli", "bench"):
        importlib.import_module(f"fedheat.{name}")
    assert sys.modules["fedheat.solver"] is solver and pkg.ExplicitEngine is fh.ExplicitEngine
    pkg.__fh_alias__ = True
    return True


_OK = os.path.isdir(VENDORED) and _install_aliases()


def pytest_ignore_collect(collection_path, config):
    # nothing to run without the vendored files (fresh clone) or the reference package
    if not _OK and "vendored" in str(collection_path):
        return True
    return None


def pytest_collection_modifyitems(config, items):
    for item in items:
        if "reference_suite" not in item.nodeid:
            continue
        item.add_marker(pytest.mark.gpu)
        for key, why in SKIPS.items():
            if key in item.nodeid:
                item.add_marker(pytest.mark.skip(reason=why))


@pytest.fixture()
def rng():
    import numpy as np

    return np.random.default_rng(1234)
