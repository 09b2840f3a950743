"""Pins of the oracle's mesh code (O1-O3): tree, 2:1 balance, Morton order, partition, neighbours.

The paper's own multilevel mesh is the headline pin; the rest are
brute-force geometric checks on random refinements.
"""
import itertools
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_paper_mesh_level_counts(oracle_mod):
    ex = json.load(open(os.path.join(GOLD, "paper_mesh_counts.json")))
    for bc in (oracle_mod.PERIODIC, oracle_mod.OUTFLOW):
        m = oracle_mod.Mesh(mesh_nx=ex["mesh_nx"], block_nx=ex["block_nx"], max_level=ex["max_level"],
                            refinement=oracle_mod.REF_STATIC, regions=[ex["region"]],
                            bc_inner=(bc,) * 3, bc_outer=(bc,) * 3)
        assert m.level_counts(4) == ex["level_counts"]
        assert m.num_blocks() == sum(ex["level_counts"])


def test_single_block_periodic_26_self_neighbors(oracle_mod):
    m = oracle_mod.Mesh(mesh_nx=(8, 8, 8), block_nx=(8, 8, 8))
    nb = m.neighbors(0)
    assert len(nb) == 26 and all(e["gid"] == 0 and e["dlevel"] == 0 for e in nb)


def test_2x2_periodic_east_neighbor(oracle_mod):
    m = oracle_mod.Mesh(mesh_nx=(8, 8, 4), block_nx=(4, 4, 4))
    blocks = {b["lx"]: b["gid"] for b in m.blocks()}
    east = [e for e in m.neighbors(blocks[(0, 0, 0)]) if e["off"] == (1, 0, 0)]
    assert len(east) == 1 and east[0]["gid"] == blocks[(1, 0, 0)]


def test_bad_tiling_rejected(oracle_mod):
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.Mesh(mesh_nx=(30, 32, 32), block_nx=(16, 16, 16))


def test_gid_is_morton_order_and_partition(oracle_mod):
    m = oracle_mod.Mesh(mesh_nx=(64, 32, 32), block_nx=(8, 8, 8), nranks=3)
    bl = m.blocks()
    keys = [oracle_mod.morton_key(b["level"], b["lx"], 0) for b in bl]
    assert keys == sorted(keys) and len(set(keys)) == len(keys)
    ranks = [b["rank"] for b in bl]
    assert ranks == sorted(ranks)
    n = len(bl)
    for r in range(3):
        lo, hi = oracle_mod.partition(n, 3, r)
        assert ranks[lo:hi] == [r] * (hi - lo)


@pytest.mark.parametrize("R,root", [(1, (4, 4, 4)), (2, (8, 4, 4)), (4, (8, 8, 4)), (8, (8, 8, 8))])
def test_weak_config_partition_is_4cubed_cube(oracle_mod, R, root):
    """contiguous Morton ranges give every rank a 4x4x4 cube of blocks."""
    m = oracle_mod.Mesh(mesh_nx=tuple(4 * r for r in root), block_nx=(4, 4, 4), nranks=R)
    by_rank = {}
    for b in m.blocks():
        by_rank.setdefault(b["rank"], []).append(b["lx"])
    assert len(by_rank) == R
    for r, lxs in by_rank.items():
        a = np.array(lxs)
        assert len(lxs) == 64
        assert all(a[:, d].max() - a[:, d].min() == 3 for d in range(3))


# ---------------------------------------------------------------- brute force geometry
def _finest_boxes(blocks, L):
    out = []
    for b in blocks:
        s = 1 << (L - b["level"])
        out.append([(b["lx"][d] * s, (b["lx"][d] + 1) * s) for d in range(3)])
    return out


def _brute_neighbors(blocks, L, width, periodic):
    """Independent definition: B is the neighbour of A at offset o iff (a periodic image of) B
    overlaps, with positive volume, the same-level box T = A shifted by o (where A's ghosts at o
    live), and that image of B touches A."""
    boxes = np.array(_finest_boxes(blocks, L))           # [B, 3, 2]
    shifts = np.array(list(itertools.product(*[[-width[d], 0, width[d]] if periodic[d] else [0]
                                               for d in range(3)])))   # [S, 3]
    imgs = boxes[:, None, :, :] + shifts[None, :, :, None]             # [B, S, 3, 2]
    res = {}
    for a in range(len(boxes)):
        A = boxes[a]
        size = A[:, 1] - A[:, 0]
        touch = np.all((imgs[..., 0] <= A[:, 1]) & (imgs[..., 1] >= A[:, 0]), axis=-1)   # [B, S]
        s = set()
        for o in itertools.product((-1, 0, 1), repeat=3):
            if o == (0, 0, 0):
                continue
            T = A + (np.array(o) * size)[:, None]
            overlap = np.all((imgs[..., 0] < T[:, 1]) & (imgs[..., 1] > T[:, 0]), axis=-1)
            for b in np.nonzero(np.any(overlap & touch, axis=1))[0]:
                s.add((int(b), o))
        res[a] = s
    return res


def _random_mesh(oracle_mod, rng):
    root = tuple(int(x) for x in rng.integers(1, 4, size=3))
    L = int(rng.integers(1, 4))
    periodic = [bool(x) for x in rng.integers(0, 2, size=3)]
    regs = []
    for _ in range(int(rng.integers(1, 4))):
        lev = int(rng.integers(1, L + 1))
        r = []
        for d in range(3):
            a, b = sorted(rng.uniform(0, 1, 2))
            r += [a, b + 1e-3]
        regs.append([lev] + r)
    bc = [oracle_mod.PERIODIC if p else oracle_mod.OUTFLOW for p in periodic]
    m = oracle_mod.Mesh(mesh_nx=tuple(4 * r for r in root), block_nx=(4, 4, 4), max_level=L,
                        refinement=oracle_mod.REF_STATIC, regions=regs, bc_inner=bc, bc_outer=bc)
    width = [r << L for r in root]
    return m, L, width, periodic


def test_random_meshes_coverage_balance_neighbors(oracle_mod):
    rng = np.random.default_rng(20220224)
    checked = 0
    for trial in range(40):
        m, L, width, periodic = _random_mesh(oracle_mod, rng)
        bl = m.blocks()
        if len(bl) > 300:
            continue
        checked += 1
        boxes = _finest_boxes(bl, L)
        # coverage: volumes add up and no two leaves overlap
        vol = sum(np.prod([b[d][1] - b[d][0] for d in range(3)]) for b in boxes)
        assert vol == np.prod(width)
        for a in range(len(boxes)):
            for b in range(a + 1, len(boxes)):
                assert not all(boxes[a][d][0] < boxes[b][d][1] and boxes[b][d][0] < boxes[a][d][1]
                               for d in range(3))
        brute = _brute_neighbors(bl, L, width, periodic)
        for b in bl:
            nb = m.neighbors(b["gid"])
            got = {(e["gid"], e["off"]) for e in nb}
            assert len(got) == len(nb)
            assert got == brute[b["gid"]], (trial, b)
            for e in nb:
                # 2:1 balance over faces, edges and corners
                assert abs(bl[e["gid"]]["level"] - b["level"]) <= 1
                assert e["dlevel"] == bl[e["gid"]]["level"] - b["level"]
                assert e["rank"] == bl[e["gid"]]["rank"]
                # symmetry: the neighbour lists me too; same level: at the opposite offset
                back = m.neighbors(e["gid"])
                assert b["gid"] in {x["gid"] for x in back}
                if e["dlevel"] == 0:
                    assert (b["gid"], tuple(-o for o in e["off"])) in {(x["gid"], x["off"]) for x in back}
            # canonical order: offsets ascend in (o3, o2, o1) order, fine children ascend
            order = [(e["off"][2], e["off"][1], e["off"][0], e["fine"][1], e["fine"][0]) for e in nb]
            assert order == sorted(order)
    assert checked >= 20
