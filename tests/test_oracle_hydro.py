"""Pins of the oracle's time integration (O5, O6, O8, O10) against what the paper and the
mathematics fix: conservation, uniform-state preservation, mirror symmetry, Sod vs the exact
Riemann solution, second-order convergence of a linear wave, the dt worked example."""
import json
import os

import numpy as np
import pytest

import exact_riemann as ER

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _all(m):
    return np.stack([m.get_state(b) for b in range(m.num_blocks())])


# ---------------------------------------------------------------- uniform state (C-PIN)
@pytest.mark.parametrize("multilevel", [False, True])
@pytest.mark.parametrize("vel", [(0.0, 0.0, 0.0), (0.3, -0.7, 0.11)])
def test_uniform_state_stays_bitwise_uniform(oracle_mod, multilevel, vel):
    kw = dict(mesh_nx=(16, 16, 16), block_nx=(8, 8, 8))
    if multilevel:
        kw.update(max_level=1, refinement=oracle_mod.REF_STATIC, regions=[(1, 0.2, 0.45, 0.2, 0.45, 0.6, 0.8)])
    m = oracle_mod.Mesh(**kw)
    if multilevel:
        assert len(set(b["level"] for b in m.blocks())) == 2
    W = np.array([1.3, *vel, 0.9])
    U = oracle_mod.prim_to_cons(W, 5 / 3)
    n = m.num_blocks()
    for b in range(n):
        m.set_state(b, np.broadcast_to(U[:, None, None, None], (5, 8, 8, 8)))
    m.exchange()
    m.compute_dt()
    m.step(5)
    for b in range(n):
        S = m.get_state(b)
        for v in range(5):
            assert np.all(S[v] == U[v])


# ---------------------------------------------------------------- conservation (C-PIN)
def test_conservation_periodic_blast_uniform(oracle_mod):
    m = oracle_mod.Mesh(mesh_nx=(32, 32, 32), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3)
    m.set_problem(oracle_mod.BLAST, [10.0, 0.1, 0.1])
    t0 = m.totals()
    m.step(100)
    h = m.history()
    assert h.shape == (100, 7)
    mom_scale = np.sum(np.abs(_all(m)[:, 1:4])) / 32 ** 3
    assert abs(h[-1, 2] - t0[0]) <= 1e-12 * t0[0]
    assert abs(h[-1, 6] - t0[4]) <= 1e-12 * t0[4]
    assert np.all(np.abs(h[-1, 3:6] - t0[1:4]) <= 1e-12 * mom_scale)


def test_conservation_two_level_needs_flux_correction(oracle_mod):
    """On a periodic 2-level mesh mass/energy are conserved only with flux correction (O8)."""
    m = oracle_mod.Mesh(mesh_nx=(16, 16, 16), block_nx=(4, 4, 4), xmin=(-.5,) * 3, xmax=(.5,) * 3,
                        max_level=1, refinement=oracle_mod.REF_STATIC,
                        regions=[(1, -0.1, 0.1, -0.1, 0.1, -0.1, 0.1)])
    assert m.level_counts(2)[1] > 0 and m.level_counts(2)[0] > 0
    m.set_problem(oracle_mod.BLAST, [10.0, 0.1, 0.15])
    t0 = m.totals()
    m.step(30)
    t1 = m.totals()
    assert abs(t1[0] - t0[0]) <= 1e-12 * t0[0]
    assert abs(t1[4] - t0[4]) <= 1e-12 * t0[4]
    assert np.all(np.abs(t1[1:4] - t0[1:4]) <= 1e-12 * t0[4])


# ---------------------------------------------------------------- symmetry (C-PIN)
def test_blast_mirror_and_transpose_symmetry_bitwise(oracle_mod):
    n = 16
    m = oracle_mod.Mesh(mesh_nx=(2 * n,) * 3, block_nx=(n,) * 3, xmin=(-.5,) * 3, xmax=(.5,) * 3)
    m.set_problem(oracle_mod.BLAST, [10.0, 0.1, 0.2])
    m.step(20)
    # assemble the global array
    G = np.zeros((5, 2 * n, 2 * n, 2 * n))
    for b in m.blocks():
        i, j, k = b["lx"]
        G[:, k * n:(k + 1) * n, j * n:(j + 1) * n, i * n:(i + 1) * n] = m.get_state(b["gid"])
    # x mirror: rho, m2, m3, E even; m1 odd
    Gx = G[:, :, :, ::-1].copy()
    Gx[1] *= -1
    assert np.array_equal(G, Gx)
    # x <-> y transpose: swap m1, m2
    Gt = np.transpose(G, (0, 1, 3, 2)).copy()
    Gt[[1, 2]] = Gt[[2, 1]]
    assert np.array_equal(G, Gt)


# ---------------------------------------------------------------- Sod vs exact (C-PIN)
def test_exact_solver_matches_textbook_star_state():
    ex = json.load(open(os.path.join(GOLD, "sod_star_state.json")))
    _, _, _, st = ER.sample_sod_like(np.array([0.5]), 0.2, 0.5, (1, 0, 1), (0.125, 0, 0.1), 1.4)
    for k in ("p_star", "u_star", "rho_star_L", "rho_star_R", "shock_speed"):
        assert abs(st[k] - ex[k]) < 1e-7, k


def _sod_l1(oracle_mod, N, wavespeed=0):
    m = oracle_mod.Mesh(mesh_nx=(N, 4, 4), block_nx=(N // 2, 4, 4), gamma=1.4, wavespeed=wavespeed,
                        bc_inner=(oracle_mod.OUTFLOW, 0, 0), bc_outer=(oracle_mod.OUTFLOW, 0, 0))
    m.set_problem(oracle_mod.SOD, [0.5])
    m.step(100000, 0.2)
    assert abs(m.time()[0] - 0.2) < 1e-15
    rho = np.concatenate([m.get_state(b)[0, 0, 0] for b in range(m.num_blocks())])
    # y,z are periodic with uniform data: every row must be identical
    for b in range(m.num_blocks()):
        S = m.get_state(b)
        assert np.all(S[0] == S[0, :1, :1, :])
        assert np.all(S[2] == 0) and np.all(S[3] == 0)
    x = (np.arange(N) + 0.5) / N
    r, _, _, _ = ER.sample_sod_like(x, 0.2, 0.5, (1, 0, 1), (0.125, 0, 0.1), 1.4)
    return np.abs(rho - r).mean()


def test_sod_converges_to_exact_solution(oracle_mod):
    e = [_sod_l1(oracle_mod, N) for N in (64, 128, 256)]
    assert e[0] / e[1] >= 1.6 and e[1] / e[2] >= 1.6, e
    assert e[2] <= 5e-3, e


def test_sod_einfeldt_converges_to_exact_solution(oracle_mod):
    """the Einfeldt wave-speed variant (A4) on the same problem: converges to the exact Riemann
    solution at least as fast, with errors close to Davis' (the SURVEY's 1D prototype found the two
    equal to 4 digits on smooth problems)"""
    e = [_sod_l1(oracle_mod, N, oracle_mod.EINFELDT) for N in (64, 128, 256)]
    d = _sod_l1(oracle_mod, 256)
    assert e[0] / e[1] >= 1.6 and e[1] / e[2] >= 1.6, e
    assert e[2] <= 5e-3 and abs(e[2] - d) <= 0.2 * d, (e, d)


# ---------------------------------------------------------------- linear wave, 2nd order (C-PIN)
def _wave_l1(oracle_mod, N, k, thin, recon=0):
    if thin:
        mesh, blk = (N, 4, 4), (N // 2, 4, 4)
    else:
        mesh, blk = (N,) * 3, (N // 2,) * 3
    m = oracle_mod.Mesh(mesh_nx=mesh, block_nx=blk, recon=recon)
    A = 1e-6
    m.set_problem(oracle_mod.LINEAR_WAVE, [A, *k])
    T = 1.0 / np.sqrt(sum(x * x for x in k))
    m.step(100000, T)
    assert abs(m.time()[0] - T) < 1e-14
    err, cnt = 0.0, 0
    for b in m.blocks():
        U = m.get_state(b["gid"])
        c = [b["xmin"][d] + (np.arange(blk[d]) + 0.5) * (b["xmax"][d] - b["xmin"][d]) / blk[d] for d in range(3)]
        Z, Y, X = np.meshgrid(c[2], c[1], c[0], indexing="ij")
        rho = 1 + A * np.sin(2 * np.pi * (k[0] * X + k[1] * Y + k[2] * Z))
        err += np.abs(U[0] - rho).sum()
        cnt += U[0].size
    return err / cnt


def test_linear_wave_aligned_second_order(oracle_mod):
    e = [_wave_l1(oracle_mod, N, (1, 0, 0), True) for N in (32, 64, 128)]
    r = [e[0] / e[1], e[1] / e[2]]
    assert r[0] >= 2.9 and r[1] >= 3.3, (e, r)


def test_linear_wave_oblique_3d_second_order(oracle_mod):
    e = [_wave_l1(oracle_mod, N, (1, 1, 1), False) for N in (16, 32, 64)]
    r = [e[0] / e[1], e[1] / e[2]]
    # SURVEY C-PIN: minmod in 3D converges slowly at these N; ratios must increase toward 4
    assert r[0] >= 2.1 and r[1] >= 2.4 and r[1] > r[0], (e, r)


@pytest.mark.slow
def test_linear_wave_oblique_3d_second_order_cpin(oracle_mod):
    """SURVEY C-PIN as written: oblique (1,1,1) 3D wave, minmod, N = 32/64/128, ratios >= 2.4 then
    >= 2.9 (SURVEY measured 2.56, 3.11).  ~2 min of oracle time on 8 cores, so it runs with
    PH_SLOW=1; the fast test above checks the same convergence at N = 16/32/64 (reading A42)."""
    e = [_wave_l1(oracle_mod, N, (1, 1, 1), False) for N in (32, 64, 128)]
    r = [e[0] / e[1], e[1] / e[2]]
    print("oblique C-PIN", e, r)
    assert r[0] >= 2.4 and r[1] >= 2.9, (e, r)


def test_linear_wave_vl2_second_order_and_close_to_rk2(oracle_mod):
    """VL2 (NEXT 2): second order in space and time on the aligned wave; with the same PLM in both
    stages its error is within a few percent of RK2's (the SURVEY prototype: 0.5 %)"""
    def l1(N, integ):
        m = oracle_mod.Mesh(mesh_nx=(N, 4, 4), block_nx=(N // 2, 4, 4), integrator=integ)
        m.set_problem(oracle_mod.LINEAR_WAVE, [1e-6, 1, 0, 0])
        m.step(100000, 1.0)
        x = (np.arange(N) + 0.5) / N
        rho = np.concatenate([m.get_state(b)[0, 0, 0] for b in range(2)])
        return np.abs(rho - (1 + 1e-6 * np.sin(2 * np.pi * x))).mean()
    e = [l1(N, oracle_mod.VL2) for N in (32, 64, 128)]
    assert e[0] / e[1] >= 2.9 and e[1] / e[2] >= 3.3, e
    r = l1(128, oracle_mod.RK2)
    assert abs(e[2] - r) <= 0.05 * r, (e[2], r)


def test_vl2_conserves_to_roundoff(oracle_mod):
    m = oracle_mod.Mesh(mesh_nx=(32, 32, 32), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3,
                        integrator=oracle_mod.VL2)
    m.set_problem(oracle_mod.BLAST, [10.0, 0.1, 0.15])
    t0 = m.totals()
    m.step(30)
    t1 = m.totals()
    assert abs(t1[0] - t0[0]) <= 1e-13 * t0[0] and abs(t1[4] - t0[4]) <= 1e-13 * t0[4]
    assert np.all(np.abs(t1[1:4] - t0[1:4]) <= 1e-13 * t0[4])


def test_linear_wave_vanleer_converges_faster(oracle_mod):
    e = [_wave_l1(oracle_mod, N, (1, 0, 0), True, recon=oracle_mod.VANLEER) for N in (32, 64, 128)]
    assert e[1] / e[2] >= 3.6, e


def test_linear_wave_mc_second_order_and_below_minmod(oracle_mod):
    """MC (the least clipping of the three limiters) is second order and, on a smooth wave, more
    accurate than minmod at every resolution"""
    e = [_wave_l1(oracle_mod, N, (1, 0, 0), True, recon=oracle_mod.MC) for N in (32, 64, 128)]
    m = [_wave_l1(oracle_mod, N, (1, 0, 0), True) for N in (32, 64, 128)]
    assert e[1] / e[2] >= 3.3 and all(a < b for a, b in zip(e, m)), (e, m)


# ---------------------------------------------------------------- dt (O6) and totals (O10)
def test_dt_worked_example(oracle_mod):
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))["dt"]
    N = int(round(1 / ex["dx"]))
    m = oracle_mod.Mesh(mesh_nx=(N, 4, 4), block_nx=(N, 4, 4), gamma=1.4, cfl=ex["cfl"])
    # c = 1 with rho=1, p=1/gamma; v1 = 1 -> |v1| + c = 2 = max_speed
    U = oracle_mod.prim_to_cons([1.0, 1.0, 0.0, 0.0, 1.0 / 1.4], 1.4)
    m.set_state(0, np.broadcast_to(U[:, None, None, None], (5, 4, 4, N)))
    dt = m.compute_dt()
    assert abs(dt - ex["dt"]) <= 1e-15


def test_totals_of_uniform_state(oracle_mod):
    m = oracle_mod.Mesh(mesh_nx=(16, 8, 8), block_nx=(8, 8, 8), xmax=(2.0, 1.0, 0.5))
    U = np.array([1.5, 0.25, 0.0, -1.0, 3.0])
    for b in range(m.num_blocks()):
        m.set_state(b, np.broadcast_to(U[:, None, None, None], (5, 8, 8, 8)))
    np.testing.assert_allclose(m.totals(), U * 1.0, rtol=1e-15)   # volume 2*1*0.5 = 1


def test_tlim_caps_last_step(oracle_mod):
    m = oracle_mod.Mesh(mesh_nx=(16, 16, 16), block_nx=(8, 8, 8))
    m.set_problem(oracle_mod.LINEAR_WAVE, [1e-6, 1, 0, 0])
    m.step(1000, 0.05)
    h = m.history()
    assert h[-1, 0] == 0.05
    assert np.all(np.diff(h[:, 0]) > 0)
    assert h[-1, 1] <= h[-2, 1]


@pytest.mark.parametrize("integ", [0, 1])
def test_stage_two_is_second_order_in_time(oracle_mod, integ):
    """RK2 (Heun, A1) and VL2 (midpoint predictor-corrector, NEXT 2) on a small-amplitude wave:
    halving dt at a fixed mesh cuts the time error by ~4 (second order in time); a first-order
    integrator (forward Euler, or VL2 with a wrong predictor weight) would give ~2."""
    def run(cfl):
        m = oracle_mod.Mesh(mesh_nx=(32, 4, 4), block_nx=(16, 4, 4), cfl=cfl, integrator=integ)
        m.set_problem(oracle_mod.LINEAR_WAVE, [1e-6, 1, 0, 0])
        m.step(100000, 0.25)
        return np.concatenate([m.get_state(b)[0, 0, 0] for b in range(2)])
    ref = run(0.0125)
    e1 = np.abs(run(0.2) - ref).mean()
    e2 = np.abs(run(0.1) - ref).mean()
    assert e1 / e2 > 3.0, (e1, e2)


# ---------------------------------------------------------------- Kelvin-Helmholtz (NEXT 4, A36)
def test_kh_quarter_shift_mirror_invariance(oracle_mod):
    """The KH state is invariant under T = (x -> x + L/4) o (y -> L - y, vy -> -vy); the Euler
    equations (and the scheme, bitwise: see the blast mirror test) are equivariant under both, so
    the solution stays T-invariant up to the ~2e-17 rounding of sin/exp at mirrored cell centres
    in the initial state.  An index or sign slip would show up at the 1e-2 level of vy."""
    n = 16
    m = oracle_mod.Mesh(mesh_nx=(4 * n, 4 * n, 4), block_nx=(n, n, 4), gamma=1.4)
    m.set_problem(oracle_mod.KH, [0.01, 0.05])

    def glob():
        G = np.zeros((5, 4, 4 * n, 4 * n))
        for b in m.blocks():
            i, j, _ = b["lx"]
            G[:, :, j * n:(j + 1) * n, i * n:(i + 1) * n] = m.get_state(b["gid"])
        return G
    for cycles in (0, 15):
        m.step(cycles)
        G = glob()
        T = np.roll(G[:, :, ::-1, :], n, axis=3).copy()
        T[2] *= -1
        assert np.abs(G - T).max() <= 1e-14, (cycles, np.abs(G - T).max())
    t = m.history()
    assert abs(t[-1, 2] - t[0, 2]) <= 1e-14 * t[0, 2]
