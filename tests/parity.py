"""Parity metric of SURVEY §8(c) c.3 (reading A27), shared by the GPU tests and smoke().

rho and E: |g - o| <= tol * |o|.  Momenta: |g - o| <= tol * max(|o|, M) where M is the largest
momentum magnitude of the oracle state (momenta are identically 0 or cross 0 in Sod / blast).
"""
import numpy as np

TOL = 1e-12  # north_star: max relative error 1e-12 per cell after 10 cycles


def errors(g, o):
    g = np.asarray(g)
    o = np.asarray(o)
    assert g.shape == o.shape
    M = np.abs(o[:, 1:4]).max() if o.ndim == 5 else np.abs(o[1:4]).max()
    out = {}
    for v in range(5):
        gv = g[:, v] if o.ndim == 5 else g[v]
        ov = o[:, v] if o.ndim == 5 else o[v]
        if v in (0, 4):
            den = np.abs(ov)
        else:
            den = np.maximum(np.abs(ov), M if M > 0 else 1.0)
        out[v] = float(np.max(np.abs(gv - ov) / den)) if ov.size else 0.0
    return out


def assert_parity(g, o, tol=TOL):
    e = errors(g, o)
    assert max(e.values()) <= tol, e
    return e


def gather(mesh):
    return np.stack([mesh.get_state(b) for b in range(mesh.num_blocks())])
