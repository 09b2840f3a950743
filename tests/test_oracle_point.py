"""Pins of the oracle's point functions against closed forms and worked examples.

Each check is chosen so that a plausible slip in the oracle (dropped term, wrong
sign, swapped index) fails: see DESIGN.md "Oracle pins".
"""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ cons <-> prim (a2)
def test_cons_to_prim_worked_example(oracle_mod):
    ex = gold("spec_examples.json")["cons_to_prim"]
    W, rc = oracle_mod.cons_to_prim(ex["U"], ex["gamma"])
    assert rc == 0
    # (1.4 - 1) is 0.39999999999999991 in binary64, so p lands one ulp below 1
    np.testing.assert_allclose(W, ex["W"], rtol=3e-16, atol=0)


def test_cons_to_prim_hand_computed_moving_state(oracle_mod):
    # rho=2, v=(1,2,3), p=1.5, gamma=1.4: m=(2,4,6), E = 1.5/0.4 + 0.5*2*14 = 17.75 (by hand)
    U = np.array([2.0, 2.0, 4.0, 6.0, 17.75])
    W, rc = oracle_mod.cons_to_prim(U, 1.4)
    assert rc == 0
    np.testing.assert_allclose(W, [2.0, 1.0, 2.0, 3.0, 1.5], rtol=1e-15, atol=0)
    np.testing.assert_allclose(oracle_mod.prim_to_cons([2.0, 1.0, 2.0, 3.0, 1.5], 1.4), U, rtol=1e-15)


def test_cons_prim_round_trip_random(oracle_mod):
    rng = np.random.default_rng(20220224)
    for _ in range(2000):
        W = np.array([rng.uniform(0.1, 10), *rng.normal(0, 3, 3), rng.uniform(0.01, 10)])
        U = oracle_mod.prim_to_cons(W, 5 / 3)
        W2, rc = oracle_mod.cons_to_prim(U, 5 / 3)
        assert rc == 0
        scale = np.array([W[0], *(np.abs(W[1:4]).max() + np.sqrt(W[4] / W[0]),) * 3, W[4]])
        # p is a difference E - ke: its error is relative to E, not p (S:751 asks 1e-14 rel)
        tol = np.array([1e-15, 1e-14, 1e-14, 1e-14, 1e-14 * U[4] / W[4]])
        assert np.all(np.abs(W2 - W) <= tol * np.maximum(scale, 1e-300) + 1e-300)


def test_cons_to_prim_rejects_nonpositive(oracle_mod):
    assert oracle_mod.cons_to_prim([0.0, 0, 0, 0, 1.0], 1.4)[1] != 0
    # E below kinetic energy: rho=1, m=2, E=1 -> p = 0.4*(1-2) < 0
    assert oracle_mod.cons_to_prim([1.0, 2.0, 0, 0, 1.0], 1.4)[1] != 0


# ------------------------------------------------------------------ PLM (a3)
@pytest.mark.parametrize("key", ["plm_linear", "plm_extremum", "plm_constant"])
def test_plm_worked_examples(oracle_mod, key):
    ex = gold("spec_examples.json")[key]
    ql, qr = oracle_mod.plm(*ex["q"])
    assert (ql, qr) == tuple(ex["faces"])


def test_plm_minmod_picks_smaller_slope_and_sign(oracle_mod):
    assert oracle_mod.plm(1.0, 2.0, 4.0) == (1.5, 2.5)      # min(1,2)=1
    assert oracle_mod.plm(4.0, 2.0, 1.0) == (2.5, 1.5)      # decreasing: slope -1
    assert oracle_mod.plm(0.0, 2.0, 2.5) == (1.75, 2.25)    # min(2, 0.5)
    assert oracle_mod.plm(0.0, 0.0, 5.0) == (0.0, 0.0)      # one-sided zero -> 0


def test_plm_vanleer_and_mc(oracle_mod):
    # van Leer harmonic 2 dl dr/(dl+dr): dl=1, dr=3 -> 1.5 ; MC: min(2,6,2) = 2
    assert oracle_mod.plm(0.0, 1.0, 4.0, oracle_mod.VANLEER) == (1.0 - 0.75, 1.0 + 0.75)
    assert oracle_mod.plm(0.0, 1.0, 4.0, oracle_mod.MC) == (0.0, 2.0)


# ------------------------------------------------------------------ HLLE (a4)
def _phys_flux(W, gamma):
    """independent textbook Euler flux F(W) along the normal (Toro eq. 3.4)"""
    rho, u, v, w, p = W
    E = p / (gamma - 1) + 0.5 * rho * (u * u + v * v + w * w)
    return np.array([rho * u, rho * u * u + p, rho * u * v, rho * u * w, u * (E + p)]), \
        np.array([rho, rho * u, rho * v, rho * w, E])


def _hlle_branch(WL, WR, gamma):
    """SPEC S:763-768 three-branch HLLE with Davis speeds, written independently"""
    FL, UL = _phys_flux(WL, gamma)
    FR, UR = _phys_flux(WR, gamma)
    cl, cr = np.sqrt(gamma * WL[4] / WL[0]), np.sqrt(gamma * WR[4] / WR[0])
    SL, SR = min(WL[1] - cl, WR[1] - cr), max(WL[1] + cl, WR[1] + cr)
    if SL >= 0:
        return FL
    if SR <= 0:
        return FR
    return (SR * FL - SL * FR + SL * SR * (UR - UL)) / (SR - SL)


def test_hlle_consistency(oracle_mod):
    rng = np.random.default_rng(1)
    for _ in range(500):
        W = np.array([rng.uniform(0.1, 5), *rng.normal(0, 2, 3), rng.uniform(0.1, 5)])
        F = oracle_mod.hlle(W, W, 1.4)
        Fx, _ = _phys_flux(W, 1.4)
        scale = np.abs(Fx).max() + W[4]
        assert np.all(np.abs(F - Fx) <= 4e-16 * scale * 4)


def test_hlle_supersonic_upwind(oracle_mod):
    WL = np.array([1.0, 5.0, 0.3, -0.2, 1.0])
    WR = np.array([0.5, 4.0, 0.1, 0.0, 0.5])
    F = oracle_mod.hlle(WL, WR, 1.4)
    np.testing.assert_allclose(F, _phys_flux(WL, 1.4)[0], rtol=1e-14)
    F = oracle_mod.hlle(-WL * [-1, 1, 1, 1, -1], -WR * [-1, 1, 1, 1, -1], 1.4)  # both moving left fast
    np.testing.assert_allclose(F, _phys_flux(WR * [1, -1, -1, -1, 1], 1.4)[0], rtol=1e-14)


def test_hlle_sod_face_matches_branch_form(oracle_mod):
    WL = np.array([1.0, 0.0, 0.0, 0.0, 1.0])
    WR = np.array([0.125, 0.0, 0.0, 0.0, 0.1])
    F = oracle_mod.hlle(WL, WR, 1.4)
    np.testing.assert_allclose(F, _hlle_branch(WL, WR, 1.4), rtol=2e-15, atol=1e-16)
    # random subsonic pairs: clamped form == branch form to round-off (A5)
    rng = np.random.default_rng(2)
    for _ in range(500):
        WL = np.array([rng.uniform(0.1, 5), *rng.normal(0, 1, 3), rng.uniform(0.1, 5)])
        WR = np.array([rng.uniform(0.1, 5), *rng.normal(0, 1, 3), rng.uniform(0.1, 5)])
        Fb = _hlle_branch(WL, WR, 1.4)
        np.testing.assert_allclose(oracle_mod.hlle(WL, WR, 1.4), Fb, rtol=1e-12, atol=1e-13)


def test_hlle_mirror_antisymmetry_bitwise(oracle_mod):
    """(W_L, W_R) -> (mirror W_R, mirror W_L) negates mass, transverse momentum and energy flux (A5)."""
    rng = np.random.default_rng(3)
    mir = np.array([1, -1, 1, 1, 1.0])
    for _ in range(2000):
        WL = np.array([rng.uniform(0.1, 5), *rng.normal(0, 1, 3), rng.uniform(0.1, 5)])
        WR = np.array([rng.uniform(0.1, 5), *rng.normal(0, 1, 3), rng.uniform(0.1, 5)])
        F = oracle_mod.hlle(WL, WR, 1.4)
        G = oracle_mod.hlle(WR * mir, WL * mir, 1.4)
        assert np.array_equal(G, F * np.array([-1, 1, -1, -1, -1.0]))


def _normal_shock(M, gamma, V):
    """states on either side of a shock of Mach number M (textbook Rankine-Hugoniot relations, e.g.
    Toro eqs. 3.50-3.51) in a frame where the shock moves with speed V; the upstream gas (rho 1, p 1)
    comes from the left, so the shock is a left-facing (u - c family) wave"""
    c1 = np.sqrt(gamma)
    u1 = M * c1                                   # upstream speed relative to the shock
    r = (gamma + 1) * M * M / ((gamma - 1) * M * M + 2)
    p2 = 1.0 + 2 * gamma / (gamma + 1) * (M * M - 1)
    u2 = u1 / r
    WL = np.array([1.0, u1 + V, 0.2, -0.1, 1.0])
    WR = np.array([r, u2 + V, 0.2, -0.1, p2])
    return WL, WR


@pytest.mark.parametrize("M", [1.5, 3.0, 10.0])
@pytest.mark.parametrize("V", [-0.4, 0.0, 0.6])
def test_hlle_einfeldt_exact_at_an_isolated_shock(oracle_mod, M, V):
    """Roe's property: across a single shock the Roe-averaged speed u~ - c~ equals the shock speed, so
    the Einfeldt HLLE flux is the exact Godunov flux (F_R for a left-moving shock, F_L otherwise) --
    any slip in the sqrt(rho) weights, the enthalpy average or c~ breaks this.  Davis' speeds do not
    have the property (the flux carries numerical dissipation)."""
    g = 1.4
    WL, WR = _normal_shock(M, g, V)
    FL, UL = _phys_flux(WL, g)
    FR, UR = _phys_flux(WR, g)
    np.testing.assert_allclose(FR - FL, V * (UR - UL), rtol=1e-12, atol=1e-12)  # R-H check of the fixture
    exact = FR if V < 0 else FL
    F = oracle_mod.hlle(WL, WR, g, oracle_mod.EINFELDT)
    scale = np.abs(exact).max()
    assert np.abs(F - exact).max() <= 1e-13 * scale, (F, exact)
    D = oracle_mod.hlle(WL, WR, g, oracle_mod.DAVIS)
    if V <= 0:
        assert np.abs(D - exact).max() > 1e-6 * scale


def test_hlle_einfeldt_consistency_and_mirror(oracle_mod):
    rng = np.random.default_rng(4)
    mir = np.array([1, -1, 1, 1, 1.0])
    for _ in range(500):
        W = np.array([rng.uniform(0.1, 5), *rng.normal(0, 2, 3), rng.uniform(0.1, 5)])
        F = oracle_mod.hlle(W, W, 1.4, oracle_mod.EINFELDT)
        Fx, _ = _phys_flux(W, 1.4)
        assert np.all(np.abs(F - Fx) <= 1.6e-15 * (np.abs(Fx).max() + W[4]))
        WL = np.array([rng.uniform(0.1, 5), *rng.normal(0, 1, 3), rng.uniform(0.1, 5)])
        WR = np.array([rng.uniform(0.1, 5), *rng.normal(0, 1, 3), rng.uniform(0.1, 5)])
        F = oracle_mod.hlle(WL, WR, 1.4, oracle_mod.EINFELDT)
        G = oracle_mod.hlle(WR * mir, WL * mir, 1.4, oracle_mod.EINFELDT)
        np.testing.assert_allclose(G, F * np.array([-1, 1, -1, -1, -1.0]), rtol=1e-13, atol=1e-14)
        # the Einfeldt interval contains the Davis one: never less dissipative than Davis' bounds allow
        D = oracle_mod.hlle(WL, WR, 1.4, oracle_mod.DAVIS)
        assert np.all(np.isfinite(F)) and np.all(np.isfinite(D))


# ------------------------------------------------------------------ restriction / prolongation (A10, A11)
def test_restrict_examples(oracle_mod):
    ex = gold("spec_examples.json")["restrict_pair"]
    assert oracle_mod.restrict8([1.0, 3.0] * 4) == ex["coarse"]
    assert oracle_mod.restrict8([7.25] * 8) == 7.25
    # linear field a + b.x at child centres (offsets +-1/4) -> value at the parent centre
    vals = [1.0 + 0.5 * (ci - 0.5) + 2.0 * (cj - 0.5) - 1.0 * (ck - 0.5)
            for ck in (0, 1) for cj in (0, 1) for ci in (0, 1)]
    assert oracle_mod.restrict8(vals) == 1.0


def test_restrict_uniform_bitwise_pairwise(oracle_mod):
    rng = np.random.default_rng(4)
    for x in rng.uniform(-1e3, 1e3, 5000):
        assert oracle_mod.restrict8([x] * 8) == x


def test_prolong_examples(oracle_mod):
    out = oracle_mod.prolong(2.0, [2.0] * 3, [2.0] * 3)
    assert np.all(out == 2.0)
    # linear: C=1, C-1 = 0, C+1 = 2 along x only -> children 0.75 / 1.25
    out = oracle_mod.prolong(1.0, [0.0, 1.0, 1.0], [2.0, 1.0, 1.0])
    assert np.array_equal(out, np.array([0.75, 1.25] * 4))
    # full linear in 3 dims with slopes (1, 2, -4)
    out = oracle_mod.prolong(10.0, [9.0, 8.0, 14.0], [11.0, 12.0, 6.0])
    exp = [10.0 + 0.25 * (2 * ci - 1) * 1 + 0.25 * (2 * cj - 1) * 2 + 0.25 * (2 * ck - 1) * -4
           for ck in (0, 1) for cj in (0, 1) for ci in (0, 1)]
    assert np.array_equal(out, np.array(exp))
    # extremum -> copy
    out = oracle_mod.prolong(3.0, [1.0, 1.0, 1.0], [1.0, 1.0, 1.0])
    assert np.all(out == 3.0)
    # restrict(prolong(c)) == c to round-off (A11)
    rng = np.random.default_rng(5)
    for _ in range(1000):
        c = rng.normal()
        o = oracle_mod.prolong(c, rng.normal(size=3), rng.normal(size=3))
        assert abs(oracle_mod.restrict8(o) - c) <= 4e-16 * max(1, abs(c))


# ------------------------------------------------------------------ Morton / partition / sums
def test_morton_examples(oracle_mod):
    for lev, lx, L, key in gold("spec_examples.json")["morton"]["cases"]:
        assert oracle_mod.morton_key(lev, lx, L) == key
    # bit interleave by hand: lx=(5,3,6) level 3 = (101,011,110): bits b0:(1,1,0)->0b011,
    # b1:(0,1,1)->0b110, b2:(1,0,1)->0b101  => 0b101_110_011
    assert oracle_mod.morton_key(3, (5, 3, 6), 3) == 0b101110011
    # level scaling: (level 1, 1,0,0) with max_level 2 -> X=(2,0,0) -> bit 3
    assert oracle_mod.morton_key(1, (1, 0, 0), 2) == 8


def test_partition_examples(oracle_mod):
    for nb, R, sizes in gold("spec_examples.json")["partition"]["cases"]:
        got = []
        for r in range(R):
            lo, hi = oracle_mod.partition(nb, R, r)
            got.append(hi - lo)
        assert got == sizes
    # contiguous cover
    for nb in range(0, 40):
        for R in range(1, 9):
            spans = [oracle_mod.partition(nb, R, r) for r in range(R)]
            assert spans[0][0] == 0 and spans[-1][1] == nb
            assert all(spans[i][1] == spans[i + 1][0] for i in range(R - 1))
            sz = [b - a for a, b in spans]
            assert max(sz) - min(sz) <= 1 and sz == sorted(sz, reverse=True)


def test_pairwise_sum(oracle_mod):
    assert oracle_mod.pairwise_sum(np.arange(1, 101, dtype=float)) == 5050.0
    a = np.full(1000, 0.1)
    # pairwise of equal values is exact up to a few ulps; sequential accumulates more
    assert abs(oracle_mod.pairwise_sum(a) - 100.0) < 1e-13
