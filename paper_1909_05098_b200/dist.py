"""Multi-GPU domain decomposition (one process per GPU).

The mesh is cut into ``n_domains`` domains (recursive coordinate bisection or
slabs along ``slab_axis``), each domain into tiles; rank r of W owns domains
[r D/W, (r+1) D/W).  The tile decomposition does not depend on W, and every
rank exchanges halo *temperatures* (bitwise copies) after each step, so the
result is bitwise identical for 1, 2, 4 or 8 GPUs.  Inside fh_step the halo
send/recv (NCCL, one grouped Send/Recv per neighbour on a comm stream)
overlaps the interior tiles of the next step.

`Plan` exposes the same bookkeeping without a GPU (used by the CPU tests);
`make_engine` builds a rank's engine and bootstraps NCCL through
torch.distributed (the plumbing: only the 128-byte NCCL id is broadcast).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .errors import ConfigError
from .solver import BoundarySpec, ExplicitEngine, native_inputs, resolve_boundary

DEFAULT_DOMAINS = 8


def domain_range(rank: int, world: int, n_domains: int = DEFAULT_DOMAINS):
    if world < 1 or n_domains % world:
        raise ConfigError(f"{n_domains} domains cannot be split over {world} ranks")
    w = n_domains // world
    return rank * w, (rank + 1) * w


class Plan:
    """Host-only tile / domain / halo bookkeeping of one rank (no GPU)."""

    INFO = ("n_parts", "rank_parts", "boundary_parts", "n_peers", "n_send", "n_recv", "node_lo", "node_hi",
            "corner_unique", "max_phase_tet", "max_phase_hex", "n_slots", "max_local_nodes", "colored_ok",
            "max_colors", "max_nph_tet", "max_nph_hex", "sum_nph_tet", "nph_len_tet", "sum_nph_hex", "nph_len_hex",
            "rank_slots", "rank_real_slots", "rank_local_nodes", "rank_owned_nodes", "rank_step_bytes",
            "rank_device_bytes")

    def __init__(self, mesh, material, boundary: BoundarySpec | None = None, *, world: int = 1, rank: int = 0,
                 n_domains: int = DEFAULT_DOMAINS, slab_axis: int = -1, part_nodes: int = 0, precision: int = 32,
                 robin=(), tuning=None):
        self.mesh = mesh
        self.boundary = resolve_boundary(boundary or BoundarySpec(), mesh)
        fm, fb, fo, keep, _ = native_inputs(mesh, self.boundary, [material], robin=robin, precision=precision,
                                            assembly="tiled", part_nodes=part_nodes, n_domains=n_domains,
                                            domains=domain_range(rank, world, n_domains), slab_axis=slab_axis,
                                            tuning=tuning)
        self._keep = keep
        h = C.c_void_p()
        N.check(N.lib().fh_plan_create(C.byref(fm), C.byref(fb), C.byref(fo), world, rank, C.byref(h)))
        self._h = h
        self._L = N.lib()
        info = np.zeros(len(self.INFO), np.int64)
        N.check(self._L.fh_plan_info(h, N.ptr(info, N.i64p), info.size))
        self.info = dict(zip(self.INFO, (int(v) for v in info)))
        V = mesh.n_nodes
        self.new_to_old = np.empty(V, np.int64)
        self.part_node_start = np.empty(self.info["n_parts"] + 1, np.int64)
        npeer = self.info["n_peers"]
        self.peers = np.empty(npeer, np.int32)
        self.send_offs = np.empty(npeer + 1, np.int64)
        self.recv_offs = np.empty(npeer + 1, np.int64)
        self.send_nodes = np.empty(self.info["n_send"], np.int64)
        self.recv_nodes = np.empty(self.info["n_recv"], np.int64)
        N.check(self._L.fh_plan_arrays(h, N.ptr(self.new_to_old, N.i64p), N.ptr(self.part_node_start, N.i64p),
                                       N.ptr(self.peers, N.i32p), N.ptr(self.send_offs, N.i64p),
                                       N.ptr(self.send_nodes, N.i64p), N.ptr(self.recv_offs, N.i64p),
                                       N.ptr(self.recv_nodes, N.i64p)))

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.fh_plan_destroy(self._h)
            self._h = None

    @property
    def owned_nodes(self) -> np.ndarray:
        """Original ids of the nodes this rank owns (new-order range)."""
        return self.new_to_old[self.info["node_lo"]:self.info["node_hi"]]

    def send_to(self, peer: int) -> np.ndarray:
        q = int(np.nonzero(self.peers == peer)[0][0])
        return self.send_nodes[self.send_offs[q]:self.send_offs[q + 1]]

    def recv_from(self, peer: int) -> np.ndarray:
        q = int(np.nonzero(self.peers == peer)[0][0])
        return self.recv_nodes[self.recv_offs[q]:self.recv_offs[q + 1]]


class HostTransport:
    """fh_transport over torch.distributed point-to-point on host tensors (any
    backend with send/recv, e.g. gloo): the engine packs its halo on the
    device, this exchanges the packed values with every peer, the engine
    unpacks them -- fh_step's NCCL schedule with a blocking host exchange."""

    def __init__(self):
        self._ex = N.EXCHANGE_FN(self._exchange)
        self._red = N.ALLREDUCE_FN(self._allreduce)
        self.struct = N.FhTransport(None, self._ex, self._red)
        self.error = None

    def _exchange(self, ctx, n_peers, peers, send, send_offs, recv, recv_offs, elem_bytes):
        try:
            import torch
            import torch.distributed as dist

            ct, tt = (C.c_float, torch.float32) if elem_bytes == 4 else (C.c_double, torch.float64)
            so = [send_offs[q] for q in range(n_peers + 1)]
            ro = [recv_offs[q] for q in range(n_peers + 1)]
            sbuf = np.ctypeslib.as_array(C.cast(send, C.POINTER(ct)), shape=(max(so[-1], 1),))
            rbuf = np.ctypeslib.as_array(C.cast(recv, C.POINTER(ct)), shape=(max(ro[-1], 1),))
            reqs, outs = [], []
            for q in range(n_peers):
                p = int(peers[q])
                st = torch.from_numpy(sbuf[so[q]:so[q + 1]].copy())
                rt = torch.empty(ro[q + 1] - ro[q], dtype=tt)
                reqs += [dist.isend(st, p), dist.irecv(rt, p)]
                outs.append((q, rt))
            for r in reqs:
                r.wait()
            for q, rt in outs:
                rbuf[ro[q]:ro[q + 1]] = rt.numpy()
            return 0
        except Exception as ex:  # noqa: BLE001 -- reported through the engine's status
            self.error = ex
            return 1

    def _allreduce(self, ctx, value):
        try:
            import torch
            import torch.distributed as dist

            # u64 min through an order-preserving shift into int64
            t = torch.tensor([int(value[0]) - 2**63], dtype=torch.int64)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            value[0] = int(t.item()) + 2**63
            return 0
        except Exception as ex:  # noqa: BLE001
            self.error = ex
            return 1


def make_engine(mesh, material, boundary=None, *, rank: int, world: int, device: int, n_domains=DEFAULT_DOMAINS,
                slab_axis: int = -1, attach: bool = True, transport: str = "nccl", **kwargs) -> ExplicitEngine:
    """The rank's TILED engine (its parts and their nodes only).  With
    ``attach`` the halo exchange is set up: ``transport="nccl"`` builds the
    NCCL communicator (rank 0 creates the id, torch.distributed broadcasts
    it); ``transport="host"`` attaches a HostTransport over the current
    torch.distributed process group."""
    eng = ExplicitEngine(mesh, material, boundary, assembly="tiled", device=device, n_domains=n_domains,
                         domains=domain_range(rank, world, n_domains), slab_axis=slab_axis, **kwargs)
    if attach and world > 1 and transport == "host":
        eng._transport = HostTransport()
        N.check(N.lib().fh_attach_transport(eng._h, C.byref(eng._transport.struct)))
        return eng
    if attach and world > 1:
        import torch
        import torch.distributed as dist

        uid = C.create_string_buffer(128)
        if rank == 0:
            N.check(N.lib().fh_nccl_unique_id(uid))
        t = torch.frombuffer(bytearray(uid.raw), dtype=torch.uint8).clone()
        if dist.get_backend() == "nccl":
            t = t.cuda(device)
        dist.broadcast(t, src=0)
        uid = C.create_string_buffer(bytes(t.cpu().numpy().tobytes()), 128)
        N.check(N.lib().fh_attach_nccl(eng._h, uid, rank, world))
    return eng


def gather_temperature(engine: ExplicitEngine) -> np.ndarray:
    """Full field on every rank: each rank contributes its owned nodes."""
    import torch
    import torch.distributed as dist

    T = engine.temperature()
    mask = engine.owned_mask()
    part = torch.from_numpy(np.where(mask, T, 0.0))
    if dist.get_backend() == "nccl":
        part = part.cuda()
    dist.all_reduce(part)
    return part.cpu().numpy()
