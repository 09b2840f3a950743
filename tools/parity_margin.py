"""Print the GPU-vs-oracle parity margins (max errors per variable) for a few cases."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O  # noqa: E402
import paper_2202_12309_b200 as P  # noqa: E402
from parity import errors, gather  # noqa: E402

CASES = {
    "wave32": (dict(mesh_nx=(32, 32, 32), block_nx=(32, 32, 32)), 0, [1e-6, 1, 1, 1], 10),
    "blast64": (dict(mesh_nx=(64, 64, 64), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3), 2, [10, .1, .15], 10),
    "sod": (dict(mesh_nx=(256, 4, 4), block_nx=(64, 4, 4), gamma=1.4, bc_inner=(1, 0, 0), bc_outer=(1, 0, 0)), 1, [0.5], 100),
    "blast2a": (dict(mesh_nx=(256,) * 3, block_nx=(64,) * 3, xmin=(-.5,) * 3, xmax=(.5,) * 3), 2, [10, .1, .1], 10),
}
for name in sys.argv[1:] or list(CASES):
    kw, prob, par, cyc = CASES[name]
    o, g = O.Mesh(**kw), P.Mesh(**kw)
    for m in (o, g):
        m.set_problem(prob, par)
        m.step(cyc)
    e = errors(gather(g), gather(o))
    print(name, {k: f"{v:.2e}" for k, v in e.items()}, "dt rel", abs(g.time()[1] - o.time()[1]) / o.time()[1], flush=True)
