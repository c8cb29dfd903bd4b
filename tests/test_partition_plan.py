"""Tile / domain / halo bookkeeping (host only, no GPU).

The C++ partitioner (csrc/fh_partition.cpp, exposed through fh_plan_*) is
checked bit for bit against an independent numpy restatement of its rules,
and the multi-GPU halo lists are checked for symmetry and coverage.
"""

import numpy as np
import pytest

import paper_1909_05098_b200 as fh
from paper_1909_05098_b200.dist import Plan, domain_range

MAT = fh.TissueMaterial.constant(density=1060.0, specific_heat=3600.0, conductivity=0.5)
FACES = ("x0", "x1", "y0", "y1", "z0", "z1")


def restated_partition(mesh, dirichlet, robin, n_domains, target, slab_axis=-1):
    """numpy restatement: domains by RCB (or slabs), parts by RCB, nodes
    part-major ordered (class, original id); returns new_to_old, part bounds."""
    xyz = mesh.nodes
    cls = np.zeros(mesh.n_nodes, np.int64)
    cls[robin] = 1
    cls[dirichlet] = 2

    def rcb(idx, parts, out):
        if parts <= 1 or idx.size <= 1:
            out.append(idx)
            return
        ext = xyz[idx].max(axis=0) - xyz[idx].min(axis=0)
        axis = 0
        for d in (1, 2):
            if ext[d] >= ext[axis]:
                axis = d
        left = parts // 2
        mid = int(float(idx.size) * left / parts)
        order = np.lexsort((idx, xyz[idx, axis]))
        rcb(idx[order[:mid]], left, out)
        rcb(idx[order[mid:]], parts - left, out)

    allidx = np.arange(mesh.n_nodes)
    doms = []
    if n_domains > 1 and slab_axis >= 0:
        order = np.lexsort((allidx, xyz[:, slab_axis]))
        cuts = [int(float(mesh.n_nodes) * d / n_domains) for d in range(n_domains + 1)]
        doms = [order[cuts[d]:cuts[d + 1]] for d in range(n_domains)]
    else:
        rcb(allidx, n_domains, doms)
    parts = []
    for dom in doms:
        rcb(dom, max(1, -(-dom.size // target)), parts)
    new_to_old = np.concatenate([p[np.lexsort((p, cls[p]))] for p in parts])
    bounds = np.concatenate([[0], np.cumsum([p.size for p in parts])])
    return new_to_old, bounds


@pytest.mark.parametrize("kind,div,ndom,target,slab", [("hex", 9, 1, 100, -1), ("tet", 6, 2, 64, -1),
                                                      ("hex", 10, 8, 150, -1), ("hex", 12, 4, 200, 2),
                                                      ("tet", 5, 8, 40, 2)])
def test_partition_matches_restatement_bitwise(kind, div, ndom, target, slab):
    mesh = fh.jittered_cube_mesh(kind, div, 0.1, 0.2, seed=div)
    bnd = fh.BoundarySpec(dirichlet=(("z0", 37.0), ("x1", 37.0)))
    # default (no first-touch pass): the order is exactly (part, class, original id)
    plan0 = Plan(mesh, MAT, bnd, world=1, rank=0, n_domains=ndom, part_nodes=target, slab_axis=slab)
    dn = plan0.boundary.dirichlet_nodes
    n2o, bounds = restated_partition(mesh, dn, np.empty(0, np.int64), ndom, target, slab)
    assert np.array_equal(plan0.new_to_old, n2o)
    assert np.array_equal(plan0.part_node_start, bounds)
    # first-touch order: same tiles and class ranges, nodes permuted inside each class
    plan = Plan(mesh, MAT, bnd, world=1, rank=0, n_domains=ndom, part_nodes=target, slab_axis=slab,
                tuning={"first_touch": 1})
    assert np.array_equal(plan.part_node_start, bounds)
    cls = np.zeros(mesh.n_nodes, np.int64)
    cls[dn] = 2
    for p in range(len(bounds) - 1):
        a, b = plan.new_to_old[bounds[p]:bounds[p + 1]], n2o[bounds[p]:bounds[p + 1]]
        assert np.array_equal(cls[a], cls[b])  # class ranges kept
        assert np.array_equal(np.sort(a), np.sort(b))
    # same input -> same plan
    again = Plan(mesh, MAT, bnd, world=1, rank=0, n_domains=ndom, part_nodes=target, slab_axis=slab,
                 tuning={"first_touch": 1})
    assert np.array_equal(again.new_to_old, plan.new_to_old)


def test_first_touch_order_makes_batch_gathers_contiguous():
    """Structured hex tile: corner a of consecutive slots of a batch maps to
    consecutive node ids (csrc/fh_partition.cpp step 4b)."""
    mesh = fh.generate_cube_mesh("hex", 12, 0.1)
    plan = Plan(mesh, MAT, n_domains=1, part_nodes=4096, tuning={"first_touch": 1})
    assert plan.info["n_parts"] == 1
    o2n = np.empty(mesh.n_nodes, np.int64)
    o2n[plan.new_to_old] = np.arange(mesh.n_nodes)
    conn = o2n[mesh.hexes]
    # first batch of slots = the first 256 elements in min-corner order
    order = np.argsort(conn.min(axis=1), kind="stable")[:256]
    steps = np.diff(conn[order], axis=0)
    assert np.mean(steps == 1) > 0.9


def test_structured_hex_is_corner_unique_and_tets_are_coloured():
    hexm = fh.generate_cube_mesh("hex", 8, 0.1)
    assert Plan(hexm, MAT, part_nodes=100).info["corner_unique"] == 1
    tetm = fh.generate_cube_mesh("tet", 20, 0.1)
    info = Plan(tetm, MAT, part_nodes=1536).info
    assert 1 <= info["max_phase_tet"] <= 32  # ranked fallback stays within the byte encoding
    # Kuhn tets: every interior node touches 24 tets.  With 4 accumulator rows
    # a colour class may write a node 4 times -> >= 6 colours, and a 256-slot
    # batch spans one or two of them
    assert info["colored_ok"] == 1 and 6 <= info["max_colors"] <= 16
    assert info["max_nph_tet"] <= 4
    rows4 = info["sum_nph_tet"]
    # one row: one write per node and class -> >= 24 colours, more phases
    info1 = Plan(tetm, MAT, part_nodes=1536, tuning={"tet_rows": 1}).info
    assert info1["colored_ok"] == 1 and 24 <= info1["max_colors"] <= 64
    assert info1["max_nph_tet"] <= 8 and info1["sum_nph_tet"] > rows4
    hexm = fh.jittered_cube_mesh("hex", 6, 0.1, 0.1, seed=1)
    assert Plan(hexm, MAT, part_nodes=100).info["max_colors"] <= 16  # greedy: about 8-12 colours


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("slab", [-1, 2])
def test_halo_lists_symmetric_and_covering(world, slab):
    mesh = fh.jittered_cube_mesh("hex", 10, 0.1, 0.15, seed=3)
    bnd = fh.BoundarySpec(dirichlet=tuple((f, 37.0) for f in FACES if f != "z1"))
    plans = [Plan(mesh, MAT, bnd, world=world, rank=r, n_domains=8, part_nodes=120, slab_axis=slab)
             for r in range(world)]
    dirichlet = set(plans[0].boundary.dirichlet_nodes.tolist())
    owned = [set(p.owned_nodes.tolist()) for p in plans]
    assert sum(len(o) for o in owned) == mesh.n_nodes
    assert set().union(*owned) == set(range(mesh.n_nodes))
    for r, p in enumerate(plans):
        for q in p.peers.tolist():
            assert np.array_equal(p.send_to(q), plans[q].recv_from(r))
            assert set(p.send_to(q).tolist()) <= owned[r]
        # every node of every element touching an owned free node is available
        recv = set(p.recv_nodes.tolist())
        conn = mesh.hexes
        free_owned = np.zeros(mesh.n_nodes, bool)
        free_owned[list(owned[r] - dirichlet)] = True
        touching = conn[free_owned[conn].any(axis=1)]
        need = set(np.unique(touching).tolist())
        assert need <= owned[r] | recv | dirichlet
        assert not (recv & dirichlet)


def test_slabs_talk_to_z_neighbours_only():
    mesh = fh.generate_cube_mesh("hex", 15, 0.1)  # 16 node planes -> 8 slabs of 2 planes
    plans = [Plan(mesh, MAT, world=8, rank=r, n_domains=8, part_nodes=128, slab_axis=2) for r in range(8)]
    for r, p in enumerate(plans):
        assert set(p.peers.tolist()) == {q for q in (r - 1, r + 1) if 0 <= q < 8}
        z = mesh.nodes[p.owned_nodes, 2]
        assert np.unique(z).size == 2  # whole node planes per slab


def test_domain_range_validation():
    assert domain_range(3, 4, 8) == (6, 8)
    with pytest.raises(fh.ConfigError):
        domain_range(0, 3, 8)


def test_wave_fit_default_tile_count():
    """With default part_nodes and fewer than 6 waves of resident CTAs, the
    tile count is raised to fill the last wave (148 SMs x 6 tet CTAs = 888):
    70^3 Kuhn tets, 8 domains -> 888 tiles instead of 472 at 768-node tiles."""
    mesh = fh.generate_cube_mesh("tet", 70, 0.1)
    info = Plan(mesh, MAT, n_domains=8).info
    assert info["n_parts"] == 888
    assert Plan(mesh, MAT, n_domains=8, part_nodes=768).info["n_parts"] == 472
