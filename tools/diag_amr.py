"""Time breakdown of the AMR blast (BASELINE config 3) per cycle: stage kernels, exchanges, and the
rest (tag pass, host normalisation, remesh, flux correction, reductions).

    python tools/diag_amr.py [--cycles 10] [--warmup 3]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_2202_12309_b200 as P
    u = dict(xmin=(-.5,) * 3, xmax=(.5,) * 3)
    m = P.Mesh(mesh_nx=(128,) * 3, block_nx=(32,) * 3, max_level=3, refinement=2, refine_tol=0.1,
               derefine_tol=0.025, derefine_interval=8, **u)
    m.set_problem(P.BLAST, [10.0, 0.1, 0.1])
    m.step(a.warmup)
    torch.cuda.synchronize()
    rows = []
    for _ in range(a.cycles):
        nb0 = m.num_blocks()
        m.kernel_timing(True)
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        m.step(1)
        e1.record(s)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        st, ns, ex, nx = m.kernel_timing(False)
        rows.append(dict(blocks_before=nb0, blocks_after=m.num_blocks(), cycle_ms=e0.elapsed_time(e1), wall_ms=wall,
                         stage_ms=st, stage_launches=ns, exch_ms=ex, exch_launches=nx))
    for r in rows:
        print(json.dumps(r))
    tot = {k: sum(r[k] for r in rows) / len(rows) for k in ("cycle_ms", "wall_ms", "stage_ms", "exch_ms")}
    tot["other_ms"] = tot["cycle_ms"] - tot["stage_ms"] - tot["exch_ms"]
    print("MEAN " + json.dumps(tot))


if __name__ == "__main__":
    main()
