"""Domain decomposition on the GPU, emulated on one device.

Two rank engines (domains [0,4) and [4,8) of 8) run on the same GPU one after
the other; after every step the halo temperatures go through host memory
(fh_halo_export / fh_halo_import -- the same lists the NCCL path sends).
The owned fields must equal a single engine's bit for bit: the tile
decomposition does not depend on the number of ranks.
"""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

fh = pytest.importorskip("paper_1909_05098_b200")
from paper_1909_05098_b200 import _native as N  # noqa: E402
from paper_1909_05098_b200.dist import domain_range  # noqa: E402


def step(eng, n, dt):
    rep = N.FhReport()
    N.check(eng._L.fh_step(eng._h, n, dt, C.byref(rep)))


@pytest.mark.parametrize("prec,slab", [(32, -1), (64, -1), (32, 2)])
def test_two_ranks_match_single_engine_bitwise(prec, slab):
    mesh = fh.jittered_cube_mesh("hex", 14, 0.1, 0.15, seed=21)
    mat = fh.TissueMaterial(density=fh.make_constant(1060.0), specific_heat=fh.linear_law(3600.0, -0.0005, 37.0),
                            conductivity=fh.linear_law(0.5, 0.0013, 37.0), perfusion_rate=0.525,
                            blood_specific_heat=3640.0, metabolic_rate=420.0)
    bnd = fh.BoundarySpec(dirichlet=(("z0", 37.0), ("z1", 40.0)))
    src = (fh.GaussianSource(amp=5e6, sigma=0.01, x0=(0.05, 0.05, 0.05)),)
    kw = dict(precision=prec, part_nodes=200, n_domains=8, slab_axis=slab, sources=src)
    ref = fh.ExplicitEngine(mesh, mat, bnd, assembly="tiled", **kw)
    ranks = [fh.ExplicitEngine(mesh, mat, bnd, assembly="tiled", domains=domain_range(r, 2), **kw) for r in range(2)]
    info = [e.halo_info() for e in ranks]
    assert all(i["world"] == 2 and i["n_peers"] == 1 for i in info)
    assert info[0]["n_send"] == info[1]["n_recv"] and info[1]["n_send"] == info[0]["n_recv"]
    dt = 0.9 * ref.critical_dt(37.0)
    T0 = 37.0 + 3.0 * np.sin(40 * mesh.nodes[:, 0]) * np.cos(30 * mesh.nodes[:, 1])
    for e in (ref, *ranks):
        st = e.initial_state(T0)
        N.check(e._L.fh_set_temperature(e._h, N.ptr(st.temperatures), mesh.n_nodes, 0, 0.0))
    for _ in range(30):
        step(ref, 1, dt)
        for e in ranks:
            step(e, 1, dt)
        out = [e.halo_export() for e in ranks]
        ranks[0].halo_import(out[1])
        ranks[1].halo_import(out[0])
    T = ref.temperature()
    for e in ranks:
        m = e.owned_mask()
        assert np.array_equal(e.temperature()[m], T[m])


def test_nccl_one_rank_communicator():
    """The NCCL path on one GPU: libnccl is dlopen'ed, a one-rank communicator
    is built from fh_nccl_unique_id, and the per-call fail-flag all-reduce goes
    through it -- the field must equal an engine without NCCL bit for bit, and
    an unstable step must still be reported."""
    mesh = fh.jittered_cube_mesh("hex", 10, 0.1, 0.15, seed=5)
    mat = fh.TissueMaterial.constant(density=1060.0, specific_heat=3600.0, conductivity=0.5)
    bnd = fh.BoundarySpec(dirichlet=(("z0", 37.0),), heat_loads=(("center", 1.0, 0.0, 1e9),))
    kw = dict(assembly="tiled", precision=32, part_nodes=100, n_domains=8, domains=domain_range(0, 1))
    plain = fh.ExplicitEngine(mesh, mat, bnd, **kw)
    nccl = fh.ExplicitEngine(mesh, mat, bnd, **kw)
    uid = C.create_string_buffer(128)
    N.check(N.lib().fh_nccl_unique_id(uid))
    N.check(N.lib().fh_attach_nccl(nccl._h, uid, 0, 1))
    dt = 0.9 * plain.critical_dt(37.0)
    a = plain.run(37.0, steps=50, dt=dt).state.temperatures
    b = nccl.run(37.0, steps=50, dt=dt).state.temperatures
    assert np.array_equal(a, b) and a.max() > 37.0
    st = nccl.initial_state(37.0 + 0.01 * np.sin(np.arange(mesh.n_nodes)))
    with pytest.raises(fh.InstabilityError):
        for _ in range(400):
            nccl.step(st, 10.0 * dt)
