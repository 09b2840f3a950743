"""Bitwise fingerprint of a few short runs (for A/B builds that must not change results):

    PH_LIB=variants/libph_X.so python tools/state_hash.py

Prints one sha256 per case over every block's interior state and the history rows.
"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {
    "blast-32x8-tile": dict(mesh_nx=(128, 128, 64), block_nx=(32, 32, 32)),
    "blast-16x16-tile": dict(mesh_nx=(64, 64, 48), block_nx=(16, 16, 16)),
    "blast-walls-vl2": dict(mesh_nx=(64, 64, 64), block_nx=(32, 32, 32), integrator=1,
                            bc_inner=(2, 0, 1), bc_outer=(2, 0, 1)),
}


def main():
    import numpy as np
    import paper_2202_12309_b200 as P
    for name, kw in CASES.items():
        m = P.Mesh(xmin=(-.5,) * 3, xmax=(.5,) * 3, **kw)
        m.set_problem(P.BLAST, [10.0, 0.1, 0.2, 0.05, -0.03, 0.0])
        m.step(6)
        h = hashlib.sha256()
        for g in range(m.num_blocks()):
            h.update(np.ascontiguousarray(m.get_state(g)).tobytes())
        h.update(np.ascontiguousarray(m.history()).tobytes())
        print(name, h.hexdigest()[:24], flush=True)
        m.close()


if __name__ == "__main__":
    main()
