"""Pins of the oracle's ghost exchange (O7), restriction/prolongation staging and remesh (O9)."""
import itertools

import numpy as np
import pytest


def _global_from_blocks(m, root, n):
    G = np.zeros((5, root[2] * n, root[1] * n, root[0] * n))
    for b in m.blocks():
        i, j, k = b["lx"]
        G[:, k * n:(k + 1) * n, j * n:(j + 1) * n, i * n:(i + 1) * n] = m.get_state(b["gid"])
    return G


def test_periodic_ghosts_equal_wrapped_interior(oracle_mod):
    root, n, g = (3, 2, 4), 4, 2
    m = oracle_mod.Mesh(mesh_nx=tuple(r * n for r in root), block_nx=(n,) * 3)
    rng = np.random.default_rng(7)
    for b in range(m.num_blocks()):
        m.set_state_full(b, rng.normal(size=(5, n + 2 * g, n + 2 * g, n + 2 * g)))  # garbage ghosts
    m.exchange()
    G = _global_from_blocks(m, root, n)
    P = np.pad(G, ((0, 0), (g, g), (g, g), (g, g)), mode="wrap")
    for b in m.blocks():
        i, j, k = b["lx"]
        exp = P[:, k * n:k * n + n + 2 * g, j * n:j * n + n + 2 * g, i * n:i * n + n + 2 * g]
        assert np.array_equal(m.get_state_full(b["gid"]), exp)


def test_corner_buffer_is_8_cells(oracle_mod):
    """a corner buffer of a 3D block with 2 ghost zones holds 8 numbers (per variable)."""
    n, g = 4, 2
    m = oracle_mod.Mesh(mesh_nx=(3 * n,) * 3, block_nx=(n,) * 3)
    ids = {b["lx"]: b["gid"] for b in m.blocks()}
    for lx, gid in ids.items():
        m.set_state_full(gid, np.full((5, n + 2 * g, n + 2 * g, n + 2 * g), 1.0 if lx == (2, 2, 2) else 0.0))
    m.exchange()
    A = m.get_state_full(ids[(0, 0, 0)])
    assert int((A[0] == 1.0).sum()) == 8
    assert np.all(A[0, :g, :g, :g] == 1.0)


@pytest.mark.parametrize("bc", ["outflow", "reflect", "mixed"])
def test_physical_bcs(oracle_mod, bc):
    root, n, g = (2, 2, 1), 4, 2
    O = oracle_mod
    if bc == "outflow":
        bi, bo = (O.OUTFLOW,) * 3, (O.OUTFLOW,) * 3
    elif bc == "reflect":
        bi, bo = (O.REFLECT,) * 3, (O.REFLECT,) * 3
    else:
        bi, bo = (O.REFLECT, O.PERIODIC, O.OUTFLOW), (O.OUTFLOW, O.PERIODIC, O.REFLECT)
    m = O.Mesh(mesh_nx=tuple(r * n for r in root), block_nx=(n,) * 3, bc_inner=bi, bc_outer=bo)
    rng = np.random.default_rng(8)
    for b in range(m.num_blocks()):
        m.set_state_full(b, rng.normal(size=(5, n + 2 * g, n + 2 * g, n + 2 * g)))
    m.exchange()
    G = _global_from_blocks(m, root, n)
    # expected: pad dimension by dimension x1, x2, x3 (numpy axes 3, 2, 1)
    P = G
    for d, ax in ((0, 3), (1, 2), (2, 1)):
        padw = [(0, 0)] * 4
        padw[ax] = (g, g)
        if bi[d] == O.PERIODIC:
            P = np.pad(P, padw, mode="wrap")
            continue
        lo = np.pad(P, padw, mode="symmetric" if bi[d] == O.REFLECT else "edge")
        hi = np.pad(P, padw, mode="symmetric" if bo[d] == O.REFLECT else "edge")
        sl_lo = [slice(None)] * 4
        sl_lo[ax] = slice(0, g)
        sl_hi = [slice(None)] * 4
        sl_hi[ax] = slice(-g, None)
        Q = lo.copy()
        Q[tuple(sl_hi)] = hi[tuple(sl_hi)]
        if bi[d] == O.REFLECT:
            idx = list(sl_lo)
            idx[0] = 1 + d
            Q[tuple(idx)] *= -1
        if bo[d] == O.REFLECT:
            idx = list(sl_hi)
            idx[0] = 1 + d
            Q[tuple(idx)] *= -1
        P = Q
    for b in m.blocks():
        i, j, k = b["lx"]
        exp = P[:, k * n:k * n + n + 2 * g, j * n:j * n + n + 2 * g, i * n:i * n + n + 2 * g]
        assert np.array_equal(m.get_state_full(b["gid"]), exp), b


def _two_level_mesh(O, bc):
    return O.Mesh(mesh_nx=(32, 32, 32), block_nx=(8, 8, 8), max_level=1, refinement=O.REF_STATIC,
                  regions=[(1, 0.3, 0.55, 0.45, 0.8, 0.3, 0.6)], bc_inner=(bc,) * 3, bc_outer=(bc,) * 3)


def test_constant_across_level_jump(oracle_mod):
    O = oracle_mod
    for bc in (O.PERIODIC, O.OUTFLOW, O.REFLECT):
        m = _two_level_mesh(O, bc)
        assert set(b["level"] for b in m.blocks()) == {0, 1}
        c = np.array([1.25, 0.0, 0.0, 0.0, 2.5])
        for b in range(m.num_blocks()):
            m.set_state_full(b, np.broadcast_to(c[:, None, None, None], (5, 12, 12, 12)) * 1.0)
        m.exchange()
        for b in range(m.num_blocks()):
            F = m.get_state_full(b)
            for v in range(5):
                assert np.all(F[v] == c[v])


def test_linear_field_reproduced_across_level_jump(oracle_mod):
    """restriction is exact on linear data and minmod prolongation reproduces it where slopes agree."""
    O = oracle_mod
    m = _two_level_mesh(O, O.OUTFLOW)
    coef = np.array([[1.0, 0.3, -0.2, 0.5], [0.1, -0.4, 0.25, 0.7], [2.0, 0.05, 0.6, -0.3],
                     [-1.0, 0.2, 0.2, 0.2], [3.0, -0.6, 0.1, 0.9]])
    n, g = 8, 2
    for b in m.blocks():
        dx = [(b["xmax"][d] - b["xmin"][d]) / n for d in range(3)]
        c = [b["xmin"][d] + (np.arange(-g, n + g) + 0.5) * dx[d] for d in range(3)]
        Z, Y, X = np.meshgrid(c[2], c[1], c[0], indexing="ij")
        F = np.stack([a[0] + a[1] * X + a[2] * Y + a[3] * Z for a in coef])
        F[:, g:-g, g:-g, g:-g] += 0.0
        garbage = np.where(np.pad(np.zeros((n, n, n), bool), g, constant_values=True), 1e30, 1.0)
        m.set_state_full(b["gid"], np.where(garbage == 1e30, 1e30, F))
    m.exchange()
    checked = 0
    for b in m.blocks():
        dx = [(b["xmax"][d] - b["xmin"][d]) / n for d in range(3)]
        c = [b["xmin"][d] + (np.arange(-g, n + g) + 0.5) * dx[d] for d in range(3)]
        Z, Y, X = np.meshgrid(c[2], c[1], c[0], indexing="ij")
        exp = np.stack([a[0] + a[1] * X + a[2] * Y + a[3] * Z for a in coef])
        got = m.get_state_full(b["gid"])
        # stay 3 coarse cells away from the physical boundary where outflow breaks linearity
        margin = 3 * (1.0 / 32) * 2
        ok = ((X > margin) & (X < 1 - margin) & (Y > margin) & (Y < 1 - margin) & (Z > margin) & (Z < 1 - margin))
        assert np.all(np.abs(got - exp)[:, ok] <= 1e-13), b
        if b["level"] == 1 and any(e["dlevel"] == -1 for e in m.neighbors(b["gid"])):
            ghost = np.pad(np.zeros((n, n, n), bool), g, constant_values=True)
            checked += int((ok & ghost).sum())    # prolongated ghost cells
    assert checked > 1000, checked


def test_multilevel_periodic_ghosts_are_finite(oracle_mod):
    """every ghost cell of every block (incl. corners) is written by the exchange"""
    O = oracle_mod
    m = _two_level_mesh(O, O.PERIODIC)
    for b in range(m.num_blocks()):
        F = np.full((5, 12, 12, 12), np.nan)
        F[:, 2:-2, 2:-2, 2:-2] = 1.0
        m.set_state_full(b, F)
    m.exchange()
    for b in range(m.num_blocks()):
        assert np.all(np.isfinite(m.get_state_full(b)))


# ---------------------------------------------------------------- AMR (O9)
def test_amr_blast_prerefinement_and_balance(oracle_mod):
    O = oracle_mod
    m = O.Mesh(mesh_nx=(32, 32, 32), block_nx=(8, 8, 8), xmin=(-.5,) * 3, xmax=(.5,) * 3, max_level=2,
               refinement=O.REF_ADAPTIVE, refine_tol=0.1, derefine_tol=0.025, derefine_interval=2)
    m.set_problem(O.BLAST, [10.0, 0.1, 0.1])
    lc = m.level_counts(3)
    assert lc[2] > 0, lc
    # the blocks containing the blast edge are at the finest level
    for b in m.blocks():
        inside = all(b["xmin"][d] < 0.1 and b["xmax"][d] > -0.1 for d in range(3))
        if inside:
            assert b["level"] >= 1
        for e in m.neighbors(b["gid"]):
            assert abs(e["dlevel"]) <= 1
    t0 = m.totals()
    m.step(8)
    t1 = m.totals()
    assert abs(t1[0] - t0[0]) <= 1e-12 * t0[0]
    assert abs(t1[4] - t0[4]) <= 1e-12 * t0[4]
    flags = m.refine_flags()
    assert set(np.unique(flags)) <= {-1, 0, 1}


def test_derefinement_gate(oracle_mod):
    """A16: derefinement only when cycle % derefine_interval == 0."""
    O = oracle_mod
    m = O.Mesh(mesh_nx=(16, 16, 16), block_nx=(4, 4, 4), max_level=1, refinement=O.REF_ADAPTIVE,
               regions=[(1, 0.3, 0.7, 0.3, 0.7, 0.3, 0.7)], derefine_interval=3)
    n0 = m.num_blocks()
    assert m.level_counts(2)[1] > 0
    U = O.prim_to_cons([1.0, 0.1, 0.0, 0.0, 1.0], 5 / 3)
    for b in range(n0):
        m.set_state(b, np.broadcast_to(U[:, None, None, None], (5, 4, 4, 4)))
    m.exchange()
    m.compute_dt()
    counts = []
    for c in range(4):
        m.step(1)
        counts.append(m.num_blocks())
        if c == 0:
            fl = m.refine_flags()
            lv = [b["level"] for b in m.blocks()]
            assert all(f == (-1 if l == 1 else 0) for f, l in zip(fl, lv))
    assert counts[0] == n0 and counts[1] == n0
    assert counts[2] == 64 and counts[3] == 64
    # uniform state survives remesh bitwise
    for b in range(m.num_blocks()):
        S = m.get_state(b)
        for v in range(5):
            assert np.all(S[v] == U[v])


def _deref_family_mesh(M, O=None):
    """120 blocks: 56 roots of 4^3 cells + the 8 families (64 level-1 blocks) of the region [0.3, 0.7]^3;
    uniform gas at rest except a pressure bump (p 1 -> 1.1) in the central 2^3 cells of one level-1
    block, which gives that block eps = 0.5 * 0.1 / 1 = 0.05 (between derefine_tol 0.01 and refine_tol
    0.5: flag 0) and leaves every other block's eps at 0 (the bump does not reach a neighbour's stencil,
    and tlim = 1e-9 keeps it in place for the one cycle)."""
    kw = dict(mesh_nx=(16, 16, 16), block_nx=(4, 4, 4), max_level=1, refinement=M.REF_ADAPTIVE,
              regions=[(1, 0.3, 0.7, 0.3, 0.7, 0.3, 0.7)], derefine_interval=1, refine_tol=0.5, derefine_tol=0.01)
    m = M.Mesh(**kw)
    O = O or M  # input states from the oracle's prim -> cons (test input, both sides get the same bytes)
    U = O.prim_to_cons([1.0, 0.0, 0.0, 0.0, 1.0], 5 / 3)
    Ub = O.prim_to_cons([1.0, 0.0, 0.0, 0.0, 1.1], 5 / 3)
    B = [b for b in m.blocks() if b["level"] == 1][0]
    for b in range(m.num_blocks()):
        S = np.array(np.broadcast_to(U[:, None, None, None], (5, 4, 4, 4)))
        if b == B["gid"]:
            S[:, 1:3, 1:3, 1:3] = Ub[:, None, None, None]
        m.set_state(b, S)
    return m, B


def test_derefinement_needs_the_whole_family(oracle_mod):
    """O9 / A15: a parent is re-formed only from all 8 of its children flagged -1; one child at flag 0
    keeps its family.  Closed form: 7 families merge, 56 + 7 + 8 = 71 blocks."""
    O = oracle_mod
    m, B = _deref_family_mesh(O)
    assert m.num_blocks() == 120 and m.level_counts(2) == [56, 64]
    m.exchange()
    m.compute_dt()
    m.step(1, 1e-9)
    fl = m.refine_flags()
    assert sorted(np.unique(fl, return_counts=True)[1].tolist()) == [57, 63]  # the 63 other children flag -1
    assert m.num_blocks() == 71 and m.level_counts(2) == [63, 8]
    kept = [b for b in m.blocks() if b["level"] == 1]
    assert {tuple(x >> 1 for x in b["lx"]) for b in kept} == {tuple(x >> 1 for x in B["lx"])}


def test_derefinement_one_level_per_remesh_and_2to1(oracle_mod):
    """A15 (2:1 over faces, edges and corners) on derefinement: a family may merge only if no leaf
    adjacent to it is finer than its children.  The level-2 region [0.3, 0.45]^3 covers root block
    (1,1,1) entirely (64 level-2 blocks); 2:1 refines its 26 root neighbours to level 1 (208 blocks);
    37 roots stay: 309.  With uniform gas and the gate open every cycle, the first remesh merges the 8
    level-2 families (their neighbours are level 1) but none of the 26 level-1 families (each touches a
    level-2 leaf): 37 + 208 + 8 = 253; the second merges all 27 level-1 families: 64."""
    O = oracle_mod
    kw = dict(mesh_nx=(16, 16, 16), block_nx=(4, 4, 4), max_level=2, refinement=O.REF_ADAPTIVE,
              regions=[(2, 0.3, 0.45, 0.3, 0.45, 0.3, 0.45)], derefine_interval=1, refine_tol=0.5,
              derefine_tol=0.01)
    m = O.Mesh(**kw)
    assert m.num_blocks() == 309 and m.level_counts(3) == [37, 208, 64]
    U = O.prim_to_cons([1.0, 0.0, 0.0, 0.0, 1.0], 5 / 3)
    for b in range(m.num_blocks()):
        m.set_state(b, np.broadcast_to(U[:, None, None, None], (5, 4, 4, 4)))
    m.exchange()
    m.compute_dt()
    m.step(1)
    assert m.num_blocks() == 253 and m.level_counts(3) == [37, 216, 0]
    m.step(1)
    assert m.num_blocks() == 64 and m.level_counts(3) == [64, 0, 0]


@pytest.mark.parametrize("axis", [0, 1])
def test_refinement_indicator_closed_form_on_a_linear_pressure(oracle_mod, axis):
    """A14: eps_B = max over the block of |grad p| / p with central differences (half the difference of
    the two neighbours, no dx).  On p = p0 + delta * i_global (rho = 1, v = 0) the difference is exact,
    so block b's indicator is delta / p at its first cell with two interior-or-neighbour sides -- the
    domain-boundary cell (outflow ghost = edge value) sees only delta / 2.  A dropped 1/2, a missing
    component or dividing by the wrong pressure fails this."""
    g, p0, d = 1.4, 1.0, 0.01
    shape = [8, 8, 8]
    shape[axis] = 24
    bc = [0, 0, 0]
    bc[axis] = oracle_mod.OUTFLOW
    m = oracle_mod.Mesh(mesh_nx=tuple(shape), block_nx=(8, 8, 8), max_level=1, refinement=oracle_mod.REF_ADAPTIVE,
                        refine_tol=1e9, derefine_tol=0.0, gamma=g, bc_inner=tuple(bc), bc_outer=tuple(bc))
    for b in m.blocks():
        lo = b["lx"][axis] * 8
        i = np.arange(8) + lo
        p = p0 + d * i
        U = np.zeros((5, 8, 8, 8))
        U[0] = 1.0
        shp = [1, 1, 1]
        shp[2 - axis] = 8
        U[4] = (p / (g - 1)).reshape(shp)
        m.set_state(b["gid"], U)
    m.exchange()
    m.tag_and_remesh()
    eps = m.indicators()
    first = {0: 1, 1: 8, 2: 16}  # first cell (global index) with a full central difference per block
    for b in m.blocks():
        want = d / (p0 + d * first[b["lx"][axis]])
        assert abs(eps[b["gid"]] - want) <= 1e-13 * want, (b, eps[b["gid"]], want)


# ------------------------------------------------------------------ method of images (bc_coarse pin)
def _mirror_pair(O, nlev, cycles, rng_seed):
    """A: [0,1] x [0,1]^2, reflecting walls in x1 (A9), periodic x2/x3, level jumps that touch
    the x1 = 0 wall.  B: [-1,1] x [0,1]^2 fully periodic with the mirror image of A's state and
    regions on x1 < 0.  A reflecting wall is a mirror plane, so A must equal B's x1 >= 0 half
    bitwise: the fine-ghost BCs, the coarse-staging BCs (bc_coarse, O7-B) and the staging geometry
    at walls (A12) are pinned by the periodic exchange, which never applies a physical BC."""
    L = nlev
    regA = [(L, 0.0, 0.2, 0.3, 0.7, 0.2, 0.6), (1, 0.7, 1.0, 0.0, 0.3, 0.5, 0.9)]
    regB = list(regA) + [(r[0], -r[2], -r[1], *r[3:]) for r in regA]
    n = 8
    A = O.Mesh(mesh_nx=(16, 16, 16), block_nx=(n,) * 3, max_level=L, refinement=O.REF_STATIC, regions=regA,
               bc_inner=(O.REFLECT, O.PERIODIC, O.PERIODIC), bc_outer=(O.REFLECT, O.PERIODIC, O.PERIODIC))
    B = O.Mesh(mesh_nx=(32, 16, 16), block_nx=(n,) * 3, xmin=(-1.0, 0.0, 0.0), xmax=(1.0, 1.0, 1.0),
               max_level=L, refinement=O.REF_STATIC, regions=regB)
    assert max(b["level"] for b in A.blocks()) == L
    rng = np.random.default_rng(rng_seed)
    bA = {(b["level"], b["lx"]): b["gid"] for b in A.blocks()}
    bB = {(b["level"], b["lx"]): b["gid"] for b in B.blocks()}
    assert len(bB) == 2 * len(bA)
    for (lev, (i, j, k)), gid in bA.items():
        W = np.stack([1.0 + 0.4 * rng.random((n, n, n)), 0.3 * rng.standard_normal((n, n, n)),
                      0.3 * rng.standard_normal((n, n, n)), 0.3 * rng.standard_normal((n, n, n)),
                      1.0 + 0.4 * rng.random((n, n, n))])
        U = np.stack([W[0], W[0] * W[1], W[0] * W[2], W[0] * W[3],
                      W[4] / (5 / 3 - 1) + 0.5 * W[0] * (W[1] ** 2 + W[2] ** 2 + W[3] ** 2)])
        A.set_state(gid, U)
        nx = 2 * 2 ** lev  # root blocks of A along x1 at this level
        B.set_state(bB[(lev, (i + nx, j, k))], U)
        M = U[:, :, :, ::-1].copy()
        M[1] *= -1.0
        B.set_state(bB[(lev, (nx - 1 - i, j, k))], M)
    for m in (A, B):
        m.exchange()
        m.compute_dt()
    assert A.compute_dt() == B.compute_dt()
    A.step(cycles)
    B.step(cycles)
    return A, B, bA, bB


@pytest.mark.parametrize("nlev", [1, 2])
def test_reflecting_wall_equals_mirrored_periodic_domain(oracle_mod, nlev):
    O = oracle_mod
    A, B, bA, bB = _mirror_pair(O, nlev, 4, 11 + nlev)
    for (lev, (i, j, k)), gid in bA.items():
        a = A.get_state(gid)
        b = B.get_state(bB[(lev, (i + 2 * 2 ** lev, j, k))])
        assert np.array_equal(a, b), (lev, i, j, k, float(np.abs(a - b).max()))
    assert A.time() == B.time()


def test_reflecting_wall_ghosts_equal_mirrored_interior(oracle_mod):
    """Right after an exchange, every ghost of A (fine ghosts at the wall and those prolongated from
    coarse staging that reaches the wall) equals the corresponding cell of B."""
    O = oracle_mod
    A, B, bA, bB = _mirror_pair(O, 2, 0, 5)
    for (lev, (i, j, k)), gid in bA.items():
        a = A.get_state_full(gid)
        b = B.get_state_full(bB[(lev, (i + 2 * 2 ** lev, j, k))])
        assert np.array_equal(a, b), (lev, i, j, k, float(np.abs(a - b).max()))
