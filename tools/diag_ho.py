import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
import paper_2202_12309_b200 as P
from parity import errors, gather
for recon in (0, 3, 4):
    for mesh, blk in (((16, 16, 16), (16, 16, 16)), ((32, 16, 16), (16, 16, 16)), ((32, 32, 32), (16, 16, 16))):
        for cyc in (0, 1, 3):
            kw = dict(mesh_nx=mesh, block_nx=blk, xmin=(-.5,) * 3, xmax=(.5,) * 3, recon=recon, nghost=3)
            o, g = O.Mesh(**kw), P.Mesh(**kw)
            for m in (o, g):
                m.set_problem(2, [10.0, 0.1, 0.15])
                m.step(cyc)
            Gg, Go = gather(g), gather(o)
            e = errors(Gg, Go)
            d = np.abs(Gg - Go)[:, 0]
            loc = np.unravel_index(np.argmax(d), d.shape)
            print(recon, mesh, cyc, "max", f"{max(e.values()):.2e}", "rho-loc (b,k,j,i)", loc,
                  "dt", g.time()[1], o.time()[1], flush=True)
