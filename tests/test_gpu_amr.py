"""GPU AMR (a9) vs the oracle: pre-refinement, tag flags, remesh (2:1, derefine gate), data
movement (prolongation / restriction), block lists and neighbour lists bit-exact, state 1e-12."""
import numpy as np
import pytest

from parity import assert_parity, gather

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available()
    from paper_2202_12309_b200 import _build
    _build.build()
    import paper_2202_12309_b200 as P
    return P


def _same_mesh(o, g):
    ob, gb = o.blocks(), g.blocks()
    assert [(b["gid"], b["level"], b["lx"]) for b in ob] == [(b["gid"], b["level"], b["lx"]) for b in gb]
    for gid in range(len(ob)):
        assert o.neighbors(gid) == g.neighbors(gid)


def _amr_pair(O, P, **extra):
    kw = dict(mesh_nx=(32, 32, 32), block_nx=(8, 8, 8), xmin=(-.5,) * 3, xmax=(.5,) * 3, max_level=2,
              refinement=P.REF_ADAPTIVE, refine_tol=0.1, derefine_tol=0.025, derefine_interval=2)
    kw.update(extra)
    return O.Mesh(**kw), P.Mesh(**kw)


def test_amr_prerefinement_matches_oracle(oracle_mod, P):
    o, g = _amr_pair(oracle_mod, P)
    for m in (o, g):
        m.set_problem(P.BLAST, [10.0, 0.1, 0.1])
    _same_mesh(o, g)
    assert len(set(b["level"] for b in g.blocks())) == 3
    assert_parity(gather(g), gather(o), 1e-15)


@pytest.mark.parametrize("bn", [8, 16])
def test_amr_blast_cycles_match_oracle(oracle_mod, P, bn):
    """bn 16: the TMA tag pass (tag2_kernel, 16 x 16 tiles) and stage2 on the multilevel mesh."""
    o, g = _amr_pair(oracle_mod, P, block_nx=(bn,) * 3)
    counts = []
    for m in (o, g):
        m.set_problem(P.BLAST, [10.0, 0.1, 0.1])
    for c in range(10):
        o.step(1)
        g.step(1)
        _same_mesh(o, g)
        assert np.array_equal(o.refine_flags(), g.refine_flags()), c
        counts.append(g.num_blocks())
        assert_parity(gather(g), gather(o))
    if bn == 8:  # (16^3 blocks: the blast stays inside the pre-refined blocks for these 10 cycles)
        assert len(set(counts)) > 1, counts      # the mesh actually changed
    ho, hg = o.history(), g.history()
    np.testing.assert_allclose(hg[:, :2], ho[:, :2], rtol=1e-12)
    np.testing.assert_allclose(hg[:, 2], ho[:, 2], rtol=1e-12)
    # conservation across remesh (prolongation / restriction are conservative, A10/A11)
    assert abs(hg[-1, 2] - hg[0, 2]) <= 1e-12 * hg[0, 2]
    assert abs(hg[-1, 6] - hg[0, 6]) <= 1e-12 * hg[0, 6]


def test_amr_derefinement_gate(oracle_mod, P):
    kw = dict(mesh_nx=(16, 16, 16), block_nx=(4, 4, 4), max_level=1, refinement=P.REF_ADAPTIVE,
              regions=[(1, 0.3, 0.7, 0.3, 0.7, 0.3, 0.7)], derefine_interval=3)
    o, g = oracle_mod.Mesh(**kw), P.Mesh(**kw)
    U = oracle_mod.prim_to_cons([1.0, 0.1, 0.0, 0.0, 1.0], 5 / 3)
    n0 = g.num_blocks()
    for m in (o, g):
        for b in range(n0):
            m.set_state(b, np.broadcast_to(U[:, None, None, None], (5, 4, 4, 4)))
    o.exchange()
    o.compute_dt()
    g.refresh()
    counts = []
    for c in range(4):
        o.step(1)
        g.step(1)
        _same_mesh(o, g)
        counts.append(g.num_blocks())
    assert counts == [n0, n0, 64, 64]
    for b in range(g.num_blocks()):
        S = g.get_state(b)
        for v in range(5):
            assert np.all(S[v] == U[v])


def test_derefinement_family_and_2to1_match_oracle(oracle_mod, P):
    """The two derefinement pins of test_oracle_exchange.py (family rule: 71 blocks; one level per
    remesh under 2:1: 309 -> 253 -> 64) on the GPU mesh (mesh.cpp normalize_flags + remesh), block lists,
    neighbour lists and flags equal to the oracle's."""
    import test_oracle_exchange as T
    o, _ = T._deref_family_mesh(oracle_mod)
    g, _ = T._deref_family_mesh(P, oracle_mod)
    o.exchange()
    o.compute_dt()
    g.refresh()
    o.step(1, 1e-9)
    g.step(1, 1e-9)
    _same_mesh(o, g)
    assert g.num_blocks() == 71
    assert np.array_equal(o.refine_flags(), g.refine_flags())
    kw = dict(mesh_nx=(16, 16, 16), block_nx=(4, 4, 4), max_level=2, refinement=P.REF_ADAPTIVE,
              regions=[(2, 0.3, 0.45, 0.3, 0.45, 0.3, 0.45)], derefine_interval=1, refine_tol=0.5,
              derefine_tol=0.01)
    o, g = oracle_mod.Mesh(**kw), P.Mesh(**kw)
    U = oracle_mod.prim_to_cons([1.0, 0.0, 0.0, 0.0, 1.0], 5 / 3)
    for m in (o, g):
        for b in range(m.num_blocks()):
            m.set_state(b, np.broadcast_to(U[:, None, None, None], (5, 4, 4, 4)))
    o.exchange()
    o.compute_dt()
    g.refresh()
    for want in (253, 64):
        o.step(1)
        g.step(1)
        _same_mesh(o, g)
        assert g.num_blocks() == want
        assert np.array_equal(o.refine_flags(), g.refine_flags())


def test_config3_amr_blast_full_size(oracle_mod, P):
    """BASELINE config 3: blast, 128^3 root grid of 32^3 blocks, 3 refinement levels, 10 cycles."""
    kw = dict(mesh_nx=(128,) * 3, block_nx=(32,) * 3, xmin=(-.5,) * 3, xmax=(.5,) * 3, max_level=3,
              refinement=P.REF_ADAPTIVE, refine_tol=0.1, derefine_tol=0.025, derefine_interval=2)
    o, g = oracle_mod.Mesh(**kw), P.Mesh(**kw)
    for m in (o, g):
        m.set_problem(P.BLAST, [10.0, 0.1, 0.1])
    _same_mesh(o, g)
    o.step(10)
    g.step(10)
    _same_mesh(o, g)
    assert np.array_equal(o.refine_flags(), g.refine_flags())
    assert_parity(gather(g), gather(o))


@pytest.mark.parametrize("adaptive", [False, True])
def test_kh_matches_oracle(oracle_mod, P, adaptive):
    """Kelvin-Helmholtz (the paper's AMR demo; A36): static two-level and adaptive."""
    kw = dict(mesh_nx=(32, 32, 8), block_nx=(8, 8, 8), gamma=1.4, max_level=1,
              regions=[(1, 0.0, 1.0, 0.2, 0.3, 0.0, 1.0)])
    if adaptive:
        kw.update(refinement=P.REF_ADAPTIVE, refine_tol=2e-3, derefine_tol=1e-4, derefine_interval=4)
    else:
        kw.update(refinement=P.REF_STATIC)
    o, g = oracle_mod.Mesh(**kw), P.Mesh(**kw)
    for m in (o, g):
        m.set_problem(P.KH, [0.01, 0.05])
    _same_mesh(o, g)
    for c in range(3):
        o.step(4)
        g.step(4)
        _same_mesh(o, g)
        assert_parity(gather(g), gather(o))
