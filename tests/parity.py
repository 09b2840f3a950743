"""Parity metric of SURVEY §8(c) c.3 with reading A27', shared by the GPU tests and smoke().

rho and E: |g - o| <= tol * |o|.
Momenta:   |g - o| <= tol * max(|o|, S) with S = max over cells of max(|m|, sqrt(rho E)).
sqrt(rho E) ~ rho c is the momentum scale at which the momentum equation's round-off lives:
its flux carries p ~ rho c^2, so reordering the arithmetic moves momentum by ~1e-16 * rho c even
where the momentum itself is tiny (the linear wave has |m| ~ A = 1e-6; Sod has m2 = m3 = 0).
"""
import json
import os

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


def diagnostics(g, o):
    """c.3's extra report per variable: the un-floored max relative error |g - o| / |o| over cells with
    o != 0 (and how many cells have o == 0 but g != 0), and the max absolute error."""
    g = np.asarray(g)
    o = np.asarray(o)
    if o.ndim == 4:
        g, o = g[None], o[None]
    out = {}
    for v in range(5):
        gv, ov = g[:, v], o[:, v]
        d = np.abs(gv - ov)
        nz = ov != 0
        out[v] = {"rel_unfloored": float(np.max(d[nz] / np.abs(ov[nz]))) if nz.any() else 0.0,
                  "zero_ref_nonzero_gpu": int(np.count_nonzero(d[~nz])),
                  "abs": float(d.max()) if d.size else 0.0}
    return out


def assert_parity(g, o, tol=TOL):
    e = errors(g, o)
    diag = diagnostics(g, o)
    log = os.environ.get("PH_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps({"test": os.environ.get("PYTEST_CURRENT_TEST", "?"), "metric": e, "diag": diag}) + "\n")
    print("parity", {v: (e[v], diag[v]["rel_unfloored"], diag[v]["abs"]) for v in range(5)})
    assert max(e.values()) <= tol, (e, diag)
    return e


def gather(mesh):
    return np.stack([mesh.get_state(b) for b in range(mesh.num_blocks())])
