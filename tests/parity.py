"""Parity metric of SURVEY §8(c) c.3 with reading A27', shared by the GPU tests and smoke().

rho and E: |g - o| <= tol * |o|.
Momenta:   |g - o| <= tol * max(|o|, S) with S = max over cells of max(|m|, sqrt(rho E)).
sqrt(rho E) ~ rho c is the momentum scale at which the momentum equation's round-off lives:
its flux carries p ~ rho c^2, so reordering the arithmetic moves momentum by ~1e-16 * rho c even
where the momentum itself is tiny (the linear wave has |m| ~ A = 1e-6; Sod has m2 = m3 = 0).
"""
import numpy as np

TOL = 1e-12  # north_star: max relative error 1e-12 per cell after 10 cycles


def momentum_scale(o):
    o = np.asarray(o)
    if o.ndim == 4:
        o = o[None]
    M = np.abs(o[:, 1:4]).max()
    S = np.sqrt(np.abs(o[:, 0] * o[:, 4])).max()
    return max(M, S)


def errors(g, o):
    g = np.asarray(g)
    o = np.asarray(o)
    assert g.shape == o.shape
    if o.ndim == 4:
        g, o = g[None], o[None]
    S = momentum_scale(o)
    out = {}
    for v in range(5):
        gv, ov = g[:, v], o[:, v]
        den = np.abs(ov) if v in (0, 4) else np.maximum(np.abs(ov), S)
        out[v] = float(np.max(np.abs(gv - ov) / den)) if ov.size else 0.0
    return out


def assert_parity(g, o, tol=TOL):
    e = errors(g, o)
    assert max(e.values()) <= tol, e
    return e


def gather(mesh):
    return np.stack([mesh.get_state(b) for b in range(mesh.num_blocks())])
