"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py [--cases all]

  wave1   config 1 (32^3 single block): stage2 kernel with the k-split, CUDA graph, dt / totals
  blast2  2 blocks of 64^3: stage2 with direct halo between blocks, both stages, H path
  smr     static 2-level mesh of 32^3 blocks: stage2 ML (flux slots), exchange phases, reflux, rfx_reduce
  amr     adaptive 3-level mesh of 8^3 blocks: the round-1 stage kernel, tag, remesh, prolong / restrict
  amr16   adaptive 3-level mesh of 16^3 blocks: stage2 ML, the TMA tag pass (tag2), remesh
  sod     thin Sod with outflow / reflect walls (16^3 blocks): physical BCs in the exchange
  ho      PPM with nghost 3: the exact-arithmetic high-order path
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {
    "wave1": (dict(mesh_nx=(32,) * 3, block_nx=(32,) * 3), 0, [1e-6, 1, 1, 1], 3),
    "blast2": (dict(mesh_nx=(128, 64, 64), block_nx=(64,) * 3, xmin=(-.5,) * 3, xmax=(.5,) * 3), 2, [10.0, 0.1, 0.2], 2),
    "smr": (dict(mesh_nx=(64,) * 3, block_nx=(32,) * 3, xmin=(-.5,) * 3, xmax=(.5,) * 3, max_level=1, refinement=1,
                 regions=[(1, -0.1, 0.1, -0.1, 0.1, -0.1, 0.1)]), 2, [10.0, 0.1, 0.1], 2),
    "amr": (dict(mesh_nx=(32,) * 3, block_nx=(8,) * 3, xmin=(-.5,) * 3, xmax=(.5,) * 3, max_level=2, refinement=2,
                 refine_tol=0.1, derefine_tol=0.025, derefine_interval=2), 2, [10.0, 0.1, 0.1], 3),
    "amr16": (dict(mesh_nx=(64,) * 3, block_nx=(16,) * 3, xmin=(-.5,) * 3, xmax=(.5,) * 3, max_level=2, refinement=2,
                   refine_tol=0.1, derefine_tol=0.025, derefine_interval=2), 2, [10.0, 0.1, 0.1], 3),
    "sod": (dict(mesh_nx=(64, 16, 16), block_nx=(16,) * 3, gamma=1.4, bc_inner=(1, 2, 0), bc_outer=(1, 2, 0)), 1,
            [0.5], 3),
    "ho": (dict(mesh_nx=(32,) * 3, block_nx=(16,) * 3, xmin=(-.5,) * 3, xmax=(.5,) * 3, recon=3, nghost=3), 2,
           [10.0, 0.1, 0.2], 2),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="all")
    a = ap.parse_args()
    import paper_2202_12309_b200 as P
    names = list(CASES) if a.cases == "all" else a.cases.split(",")
    for n in names:
        kw, prob, par, cyc = CASES[n]
        m = P.Mesh(**kw)
        m.set_problem(prob, par)
        m.step(cyc)
        t = m.time()
        m.close()
        print(f"case {n}: t={t[0]:.6g} cycle={t[2]}", flush=True)
    print("SANITIZE_CASES_DONE")


if __name__ == "__main__":
    main()
