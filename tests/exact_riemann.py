"""Exact Riemann solver for the ideal-gas Euler equations (Toro 2009, ch. 4).

Test-only, independent of the oracle: used to pin the oracle's Sod run (C-PIN "Sod").
Its star state is itself pinned against tests/golden/sod_star_state.json.
"""
import numpy as np


def _fK(p, rhoK, pK, gamma):
    cK = np.sqrt(gamma * pK / rhoK)
    if p > pK:  # shock
        A = 2.0 / ((gamma + 1) * rhoK)
        B = (gamma - 1) / (gamma + 1) * pK
        f = (p - pK) * np.sqrt(A / (p + B))
        df = np.sqrt(A / (B + p)) * (1 - (p - pK) / (2 * (B + p)))
    else:  # rarefaction
        f = 2 * cK / (gamma - 1) * ((p / pK) ** ((gamma - 1) / (2 * gamma)) - 1)
        df = 1.0 / (rhoK * cK) * (p / pK) ** (-(gamma + 1) / (2 * gamma))
    return f, df


def star_state(WL, WR, gamma):
    rl, ul, pl = WL
    rr, ur, pr = WR
    p = 0.5 * (pl + pr)
    for _ in range(100):
        fl, dfl = _fK(p, rl, pl, gamma)
        fr, dfr = _fK(p, rr, pr, gamma)
        dp = (fl + fr + (ur - ul)) / (dfl + dfr)
        p = max(p - dp, 1e-12)
        if abs(dp) < 1e-15 * p:
            break
    fl, _ = _fK(p, rl, pl, gamma)
    fr, _ = _fK(p, rr, pr, gamma)
    u = 0.5 * (ul + ur) + 0.5 * (fr - fl)
    return p, u


def sample_sod_like(x, t, x0, WL, WR, gamma):
    """Density, velocity, pressure at positions x for a left rarefaction / right shock problem."""
    rl, ul, pl = WL
    rr, ur, pr = WR
    ps, us = star_state(WL, WR, gamma)
    assert ps < pl and ps > pr, "sampler covers left-rarefaction / right-shock only"
    g = gamma
    cl = np.sqrt(g * pl / rl)
    cr = np.sqrt(g * pr / rr)
    rsl = rl * (ps / pl) ** (1 / g)
    csl = cl * (ps / pl) ** ((g - 1) / (2 * g))
    rsr = rr * ((ps / pr + (g - 1) / (g + 1)) / ((g - 1) / (g + 1) * ps / pr + 1))
    S = ur + cr * np.sqrt((g + 1) / (2 * g) * ps / pr + (g - 1) / (2 * g))
    xi = (np.asarray(x) - x0) / t
    rho = np.empty_like(xi)
    u = np.empty_like(xi)
    p = np.empty_like(xi)
    head, tail = ul - cl, us - csl
    m = xi <= head
    rho[m], u[m], p[m] = rl, ul, pl
    m = (xi > head) & (xi <= tail)
    uf = 2 / (g + 1) * (cl + (g - 1) / 2 * ul + xi[m])
    cf = 2 / (g + 1) * (cl + (g - 1) / 2 * (ul - xi[m]))
    rho[m] = rl * (cf / cl) ** (2 / (g - 1))
    u[m] = uf
    p[m] = pl * (cf / cl) ** (2 * g / (g - 1))
    m = (xi > tail) & (xi <= us)
    rho[m], u[m], p[m] = rsl, us, ps
    m = (xi > us) & (xi <= S)
    rho[m], u[m], p[m] = rsr, us, ps
    m = xi > S
    rho[m], u[m], p[m] = rr, ur, pr
    return rho, u, p, dict(p_star=ps, u_star=us, rho_star_L=rsl, rho_star_R=rsr, shock_speed=S)
