"""Two processes, one rank engine each, running fh_step's real multi-GPU
schedule through the host transport hook (fh_attach_transport over gloo).

Per step every rank runs its interior tiles, its boundary tiles, the pack
kernel, the exchange (here: device -> host, gloo point-to-point, host ->
device instead of NCCL) and the unpack kernel -- the order of the NCCL path.
Each engine holds only its own parts and the nodes they read (rank-local
numbering).  Both processes share the one GPU of the box, but no kernel waits
on another process: the exchange blocks on the host between launches.

Checks, against a single engine owning every domain (rank 0 runs it too):
* the gathered field after 40 steps is bit-identical (fp32 and fp64);
* a runaway step is reported by both ranks with the single engine's step and
  node, and the gathered field is the one right after that step (the failing
  call is replayed from its start on every rank up to the failing step).
"""

import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

WORLD = 2


def _problem():
    import paper_1909_05098_b200 as fh

    mesh = fh.jittered_cube_mesh("hex", 14, 0.1, 0.15, seed=21)
    mat = fh.TissueMaterial(density=fh.make_constant(1060.0), specific_heat=fh.linear_law(3600.0, -0.0005, 37.0),
                            conductivity=fh.linear_law(0.5, 0.0013, 37.0), perfusion_rate=0.525,
                            blood_specific_heat=3640.0, metabolic_rate=420.0)
    bnd = fh.BoundarySpec(dirichlet=(("z0", 37.0), ("z1", 40.0)))
    src = (fh.GaussianSource(amp=5e6, sigma=0.01, x0=(0.05, 0.05, 0.05)),)
    T0 = 37.0 + 3.0 * np.sin(40 * mesh.nodes[:, 0]) * np.cos(30 * mesh.nodes[:, 1])
    return fh, mesh, mat, bnd, src, T0


def _worker(rank, port, prec, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        from paper_1909_05098_b200 import _native as N
        from paper_1909_05098_b200.dist import gather_temperature, make_engine

        fh, mesh, mat, bnd, src, T0 = _problem()
        kw = dict(precision=prec, part_nodes=200, n_domains=8, sources=src)
        eng = make_engine(mesh, mat, bnd, rank=rank, world=WORLD, device=0, transport="host", **kw)
        info = eng.halo_info()
        assert info["world"] == WORLD and info["n_peers"] == 1
        lay = eng.layout()
        dt = 0.9 * eng.critical_dt(37.0)
        rep = N.FhReport()
        L, h = eng._L, eng._h
        N.check(L.fh_set_temperature(h, N.ptr(T0), mesh.n_nodes, 0, 0.0))
        N.check(L.fh_step(h, 15, dt, C.byref(rep)))
        N.check(L.fh_step(h, 25, dt, C.byref(rep)))
        T = gather_temperature(eng)
        # runaway: 4x the stable step from a rough field
        Tr = 37.0 + np.random.default_rng(2).uniform(-1, 1, mesh.n_nodes)
        N.check(L.fh_set_temperature(h, N.ptr(Tr), mesh.n_nodes, 0, 0.0))
        rc = L.fh_step(h, 300, 4.0 * dt, C.byref(rep))
        fail = (rc, rep.fail_step, rep.fail_node, rep.fail_value)
        Tf = gather_temperature(eng)
        out = {"T": T, "fail": fail, "Tf": Tf, "slots": lay["n_slots"], "owned": lay["n_nodes_owned"]}
        if rank == 0:  # the single-engine reference
            ref = fh.ExplicitEngine(mesh, mat, bnd, assembly="tiled", **kw)
            for E in (ref,):
                N.check(E._L.fh_set_temperature(E._h, N.ptr(T0), mesh.n_nodes, 0, 0.0))
                N.check(E._L.fh_step(E._h, 40, dt, C.byref(rep)))
            out["T_ref"] = ref.temperature()
            N.check(ref._L.fh_set_temperature(ref._h, N.ptr(Tr), mesh.n_nodes, 0, 0.0))
            rc = ref._L.fh_step(ref._h, 300, 4.0 * dt, C.byref(rep))
            out["fail_ref"] = (rc, rep.fail_step, rep.fail_node, rep.fail_value)
            out["Tf_ref"] = ref.temperature()
            out["slots_ref"] = ref.layout()["n_slots"]
            out["owned_ref"] = ref.layout()["n_nodes_owned"]
            out["V"] = mesh.n_nodes
        result_q.put((rank, True, out))
    except Exception as err:  # pragma: no cover - reported to the parent
        import traceback

        result_q.put((rank, False, traceback.format_exc()[-3000:] + repr(err)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("prec", [32, 64])
def test_two_process_host_transport_bitwise(prec):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + os.getpid() % 1000 + prec
    procs = [ctx.Process(target=_worker, args=(r, port, prec, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = {}
    for _ in range(WORLD):
        rank, ok, out = q.get(timeout=600)
        assert ok, f"rank {rank}: {out}"
        results[rank] = out
    for p in procs:
        p.join(timeout=60)
    r0, r1 = results[0], results[1]
    assert np.array_equal(r0["T"], r0["T_ref"]) and np.array_equal(r1["T"], r0["T_ref"])
    # each rank holds about half of the slots (the tiles are the same for any rank count)
    assert r0["slots"] + r1["slots"] == r0["slots_ref"]
    assert r0["owned"] + r1["owned"] == r0["owned_ref"]
    rc_ref, fs_ref, fn_ref, fv_ref = r0["fail_ref"]
    assert rc_ref == 2 and fs_ref > 2
    for r in (r0, r1):
        rc, fs, fn, fv = r["fail"]
        assert (rc, fs, fn) == (2, fs_ref, fn_ref)
        assert fv == fv_ref or (np.isnan(fv) and np.isnan(fv_ref))
        assert np.array_equal(r["Tf"], r0["Tf_ref"], equal_nan=True)
