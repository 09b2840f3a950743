"""Small driver for ncu captures: a 2b-shaped run (64^3 blocks, blast) on fewer blocks.

    python tools/profile_run.py --blocks-per-dim 4 --cycles 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--blocks-per-dim", type=int, default=4)
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--cycles", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_2202_12309_b200 as P
    b, n = a.blocks_per_dim, a.n
    m = P.Mesh(mesh_nx=(b * n,) * 3, block_nx=(n,) * 3, xmin=(-0.5,) * 3, xmax=(0.5,) * 3)
    m.set_problem(P.BLAST, [10.0, 0.1, 0.1])
    m.step(a.cycles)
    torch.cuda.synchronize()
    print("done", m.time())


if __name__ == "__main__":
    main()
