"""Pins of the oracle's NEXT-3 reconstructions: PPM (Colella & Woodward 1984, reading A37) and
WENO-Z (Borges et al. 2008, reading A38), nghost = 3 (A8).  The paper names neither (SURVEY §8(f):
"parity unpinned by the paper"); these pins come from their textbook definitions and properties."""
import numpy as np
import pytest


def _quad_avgs(i0, h=1.0):
    # cell averages of x^2 over [x-h/2, x+h/2] at centres i0-2 .. i0+2
    xs = (np.arange(5) - 2 + i0) * h
    return xs * xs + h * h / 12.0


@pytest.mark.parametrize("recon", [3, 4])
def test_constant_and_linear_are_exact(oracle_mod, recon):
    assert oracle_mod.recon5([3.5] * 5, recon) == (3.5, 3.5)
    ql, qr = oracle_mod.recon5([1.0, 2.0, 3.0, 4.0, 5.0], recon)
    assert abs(ql - 2.5) < 1e-15 and abs(qr - 3.5) < 1e-15
    ql, qr = oracle_mod.recon5([5.0, 4.0, 3.0, 2.0, 1.0], recon)
    assert abs(ql - 3.5) < 1e-15 and abs(qr - 2.5) < 1e-15


@pytest.mark.parametrize("recon", [3, 4])
def test_quadratic_cell_averages_give_exact_face_values(oracle_mod, recon):
    """WENO-Z: every 3-cell candidate is exact for quadratics; PPM: the 4th-order interface formula
    is exact for quadratics away from extrema (no limiting active)."""
    for i0 in (4.0, 7.0, -6.0):
        ql, qr = oracle_mod.recon5(_quad_avgs(i0), recon)
        assert abs(ql - (i0 - 0.5) ** 2) < 1e-12 and abs(qr - (i0 + 0.5) ** 2) < 1e-12, (i0, ql, qr)


def test_ppm_flattens_extrema_and_limits_overshoots(oracle_mod):
    assert oracle_mod.recon5([0.0, 1.0, 3.0, 1.0, 0.0], 3) == (3.0, 3.0)   # local maximum
    rng = np.random.default_rng(9)
    for _ in range(3000):
        q = rng.normal(size=5)
        ql, qr = oracle_mod.recon5(q, 3)
        c = q[2]
        d, m6 = qr - ql, 6 * (c - 0.5 * (ql + qr))
        # CW84 1.10: the limited parabola has no interior extremum (to round-off)
        assert d * m6 <= d * d * (1 + 1e-12) + 1e-300 and -d * d * (1 + 1e-12) - 1e-300 <= d * m6
        # face values lie within the range of the adjacent cell values
        assert min(q[1], q[2]) - 1e-12 <= ql <= max(q[1], q[2]) + 1e-12
        assert min(q[2], q[3]) - 1e-12 <= qr <= max(q[2], q[3]) + 1e-12


def test_wenoz_is_essentially_non_oscillatory_and_symmetric(oracle_mod):
    # a step inside the stencil: the right face of cell 2 follows the smooth left stencil
    ql, qr = oracle_mod.recon5([0.0, 0.0, 0.0, 1.0, 1.0], 4)
    assert abs(qr) < 1e-6 and abs(ql) < 1e-12
    rng = np.random.default_rng(10)
    for _ in range(1000):
        q = rng.normal(size=5)
        ql, qr = oracle_mod.recon5(q, 4)
        ml, mr = oracle_mod.recon5(q[::-1].copy(), 4)
        assert abs(ql - mr) <= 1e-13 * (1 + abs(ql)) and abs(qr - ml) <= 1e-13 * (1 + abs(qr))
        # affine invariance
        al, ar = oracle_mod.recon5(3.0 * q + 2.0, 4)
        assert abs(al - (3 * ql + 2)) < 1e-12 and abs(ar - (3 * qr + 2)) < 1e-12


def _wave_err(oracle_mod, N, recon, g):
    m = oracle_mod.Mesh(mesh_nx=(N, 6, 6), block_nx=(N // 2, 6, 6), recon=recon, nghost=g)
    A = 1e-6
    m.set_problem(oracle_mod.LINEAR_WAVE, [A, 1, 0, 0])
    m.step(100000, 1.0)
    err, cnt = 0.0, 0
    for b in m.blocks():
        U = m.get_state(b["gid"])
        n1 = U.shape[3]
        x = b["xmin"][0] + (np.arange(n1) + 0.5) * (b["xmax"][0] - b["xmin"][0]) / n1
        err += np.abs(U[0] - (1 + A * np.sin(2 * np.pi * x))[None, None, :]).sum()
        cnt += U[0].size
    return err / cnt


def test_high_order_linear_wave_errors(oracle_mod):
    plm = [_wave_err(oracle_mod, N, 0, 2) for N in (32, 64)]
    ppm = [_wave_err(oracle_mod, N, 3, 3) for N in (32, 64, 128)]
    wz = [_wave_err(oracle_mod, N, 4, 3) for N in (32, 64, 128)]
    # second order overall (RK2 time error), smaller constants than PLM minmod
    assert ppm[0] / ppm[1] >= 3.4 and ppm[1] / ppm[2] >= 3.4, ppm
    assert wz[0] / wz[1] >= 3.8 and wz[1] / wz[2] >= 3.8, wz
    assert ppm[1] < 0.6 * plm[1] and wz[1] < 0.1 * plm[1], (plm, ppm, wz)


def test_high_order_uniform_state_and_conservation(oracle_mod):
    for recon in (3, 4):
        m = oracle_mod.Mesh(mesh_nx=(24, 24, 24), block_nx=(12, 12, 12), xmin=(-.5,) * 3, xmax=(.5,) * 3,
                            recon=recon, nghost=3)
        m.set_problem(oracle_mod.BLAST, [10.0, 0.1, 0.2])
        t0 = m.totals()
        m.step(20)
        t1 = m.totals()
        assert abs(t1[0] - t0[0]) <= 1e-12 * t0[0] and abs(t1[4] - t0[4]) <= 1e-12 * t0[4]
        u = oracle_mod.Mesh(mesh_nx=(12, 12, 12), block_nx=(6, 6, 6), recon=recon, nghost=3)
        U = oracle_mod.prim_to_cons([1.2, 0.3, -0.1, 0.2, 0.8], 5 / 3)
        for b in range(u.num_blocks()):
            u.set_state(b, np.broadcast_to(U[:, None, None, None], (5, 6, 6, 6)))
        u.exchange()
        u.compute_dt()
        u.step(3)
        for b in range(u.num_blocks()):
            S = u.get_state(b)
            assert all(np.all(S[v] == U[v]) for v in range(5))


def test_nghost3_restrictions(oracle_mod):
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.Mesh(recon=4, nghost=2)
    with pytest.raises(oracle_mod.OracleError):
        oracle_mod.Mesh(mesh_nx=(16,) * 3, block_nx=(8,) * 3, recon=4, nghost=3, max_level=1, refinement=1,
                        regions=[(1, 0, 0.5, 0, 0.5, 0, 0.5)])
