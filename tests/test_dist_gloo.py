"""World-size-2 gloo test of the multi-GPU host path on CPU.

Each process builds its rank's plan with the native bookkeeping (no GPU),
the two ranks swap their send/recv id lists over gloo and check they agree,
then run the halo exchange protocol of fh_step (pack owned values in send
order, point-to-point exchange, unpack in recv order) on a field and check
every value a rank needs arrives bit for bit.
"""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _worker(rank, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_1909_05098_b200 as fh
        from paper_1909_05098_b200.dist import Plan

        mesh = fh.jittered_cube_mesh("hex", 9, 0.1, 0.15, seed=11)
        mat = fh.TissueMaterial.constant(density=1060.0, specific_heat=3600.0, conductivity=0.5)
        bnd = fh.BoundarySpec(dirichlet=(("z0", 37.0),))
        plan = Plan(mesh, mat, bnd, world=WORLD, rank=rank, n_domains=8, part_nodes=100)
        peer = 1 - rank
        assert plan.peers.tolist() == [peer]
        # 1. list agreement: my send list == peer's recv list (and vice versa)
        mine = torch.from_numpy(plan.send_to(peer).copy())
        n_theirs = torch.tensor([0])
        dist.send(torch.tensor([mine.numel()]), peer) if rank == 0 else dist.recv(n_theirs, peer)
        dist.recv(n_theirs, peer) if rank == 0 else dist.send(torch.tensor([mine.numel()]), peer)
        theirs = torch.empty(int(n_theirs), dtype=torch.int64)
        if rank == 0:
            dist.send(mine, peer)
            dist.recv(theirs, peer)
        else:
            dist.recv(theirs, peer)
            dist.send(mine, peer)
        assert np.array_equal(theirs.numpy(), plan.recv_from(peer))
        # 2. exchange protocol on a field known only on owned nodes
        truth = np.random.default_rng(5).standard_normal(mesh.n_nodes)
        field = np.full(mesh.n_nodes, np.nan)
        field[plan.owned_nodes] = truth[plan.owned_nodes]
        sendbuf = torch.from_numpy(field[plan.send_to(peer)].copy())
        recvbuf = torch.empty(plan.recv_from(peer).size, dtype=torch.float64)
        reqs = [dist.isend(sendbuf, peer), dist.irecv(recvbuf, peer)]
        for r in reqs:
            r.wait()
        field[plan.recv_from(peer)] = recvbuf.numpy()
        need = np.unique(plan.recv_nodes)
        assert np.array_equal(field[need], truth[need])
        result_q.put((rank, True, ""))
    except Exception as err:  # pragma: no cover - reported to the parent
        result_q.put((rank, False, repr(err)))
    finally:
        dist.destroy_process_group()


def test_two_rank_halo_protocol_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, msg in results:
        assert ok, f"rank {rank}: {msg}"


def _transport_worker(rank, port, result_q):
    """The HostTransport callbacks exactly as the engine calls them (C
    pointers to the packed send buffer, per-peer offsets, a recv buffer)."""
    import ctypes as C

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_1909_05098_b200 as fh
        from paper_1909_05098_b200.dist import HostTransport, Plan

        mesh = fh.jittered_cube_mesh("tet", 8, 0.1, 0.15, seed=3)
        mat = fh.TissueMaterial.constant(density=1060.0, specific_heat=3600.0, conductivity=0.5)
        plan = Plan(mesh, mat, world=WORLD, rank=rank, n_domains=8, part_nodes=120)
        truth = np.random.default_rng(9).standard_normal(mesh.n_nodes)
        t = HostTransport()
        for dtype, ct in ((np.float32, C.c_float), (np.float64, C.c_double)):
            send = np.ascontiguousarray(truth[plan.send_nodes].astype(dtype))
            recv = np.full(max(1, plan.recv_nodes.size), np.nan, dtype=dtype)
            peers = np.ascontiguousarray(plan.peers, dtype=np.int32)
            so = np.ascontiguousarray(plan.send_offs, dtype=np.int64)
            ro = np.ascontiguousarray(plan.recv_offs, dtype=np.int64)
            rc = t._ex(None, peers.size, peers.ctypes.data_as(C.POINTER(C.c_int32)), send.ctypes.data_as(C.c_void_p),
                       so.ctypes.data_as(C.POINTER(C.c_int64)), recv.ctypes.data_as(C.c_void_p),
                       ro.ctypes.data_as(C.POINTER(C.c_int64)), np.dtype(dtype).itemsize)
            assert rc == 0, t.error
            assert np.array_equal(recv[:plan.recv_nodes.size], truth[plan.recv_nodes].astype(dtype))
        # u64 min over ranks, including values above 2^63
        for mine in ([5, 9], [2**64 - 1, 2**64 - 2], [2**63 + 7, 3]):
            v = (C.c_uint64 * 1)(mine[rank])
            assert t._red(None, v) == 0
            assert v[0] == min(mine)
        result_q.put((rank, True, ""))
    except Exception as err:  # pragma: no cover - reported to the parent
        result_q.put((rank, False, repr(err)))
    finally:
        dist.destroy_process_group()


def test_host_transport_callbacks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_transport_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, msg in results:
        assert ok, f"rank {rank}: {msg}"
