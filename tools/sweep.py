"""Measure every BASELINE.json config on one B200 (zone-cycles/s, ms per cycle, launches per cycle).

    python tools/sweep.py [--cycles 10] [--warmup 3] [--only 1,2a,...] > profiles/r01_sweep.jsonl

Configs:
  1   linear wave, 32^3 mesh as one 32^3 block (launch-bound: CUDA graph vs eager)
  2a  blast, 256^3 mesh of 64^3 blocks (64 blocks)      2b  512^3 of 64^3 (512 blocks)
  2c  blast, 256^3 mesh of 32^3 blocks (512 blocks)
  3   blast AMR: 128^3 root, 32^3 blocks, 3 levels (remesh every cycle included in the time)
  4   256^3 cells per GPU in 64^3 blocks (the weak-scaling unit)
  5   512^3 mesh over 8 GPUs = 256^3 per GPU; block size 16^3..128^3 x pack size {all, 64, 8, 1}
Timing: CUDA events on the launch stream around `cycles` cycles after `warmup`.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

BLAST = [10.0, 0.1, 0.1]


def cases():
    c = {}
    c["1"] = dict(kw=dict(mesh_nx=(32,) * 3, block_nx=(32,) * 3), prob=0, par=[1e-6, 1, 1, 1])
    c["1-eager"] = dict(c["1"], env={"PH_NO_GRAPH": "1"})
    u = dict(xmin=(-.5,) * 3, xmax=(.5,) * 3)
    c["2a"] = dict(kw=dict(mesh_nx=(256,) * 3, block_nx=(64,) * 3, **u), prob=2, par=BLAST)
    c["2b"] = dict(kw=dict(mesh_nx=(512,) * 3, block_nx=(64,) * 3, **u), prob=2, par=BLAST)
    c["2c"] = dict(kw=dict(mesh_nx=(256,) * 3, block_nx=(32,) * 3, **u), prob=2, par=BLAST)
    c["3"] = dict(kw=dict(mesh_nx=(128,) * 3, block_nx=(32,) * 3, max_level=3, refinement=2, refine_tol=0.1,
                          derefine_tol=0.025, derefine_interval=8, **u), prob=2, par=BLAST)
    c["4"] = dict(kw=dict(mesh_nx=(256,) * 3, block_nx=(64,) * 3, **u), prob=2, par=BLAST)
    # NEXT 3: PPM / WENO-Z (nghost 3, generic high-order path, exact arithmetic)
    c["ho-ppm"] = dict(kw=dict(mesh_nx=(256,) * 3, block_nx=(64,) * 3, recon=3, nghost=3, **u), prob=2, par=BLAST)
    c["ho-wenoz"] = dict(kw=dict(mesh_nx=(256,) * 3, block_nx=(64,) * 3, recon=4, nghost=3, **u), prob=2, par=BLAST)
    c["ho-plm"] = dict(kw=dict(mesh_nx=(256,) * 3, block_nx=(64,) * 3, recon=0, nghost=3, **u), prob=2, par=BLAST)
    for r in ("ppm", "wenoz", "plm"):  # A/B: the per-face flux kernel instead of the line march
        c[f"ho-{r}-face"] = dict(c[f"ho-{r}"], env={"PH_HO_FACE": "1"})
        c[f"ho-{r}-line"] = dict(c[f"ho-{r}"], env={"PH_HO_LINE": "1"})
    # NEXT 1: the paper's own multilevel mesh: 256^3 root, 32^3 blocks, [0.3,0.7]^3 at
    # level 3 -> 296/1216/1352/21952 blocks (24,816; 813M cells; ~93 GB of block pools)
    c["nx1"] = dict(kw=dict(mesh_nx=(256,) * 3, block_nx=(32,) * 3, max_level=3, refinement=1,
                            regions=[(3, 0.3, 0.7, 0.3, 0.7, 0.3, 0.7)], xmin=(0.0,) * 3, xmax=(1.0,) * 3),
                    prob=2, par=[10.0, 0.1, 0.1, 0.5, 0.5, 0.5])
    for n in (16, 32, 64, 128):
        for ps in (0, 64, 8, 1):
            nb = (256 // n) ** 3
            if ps and ps >= nb:
                continue
            c[f"5-b{n}-p{ps or 'all'}"] = dict(kw=dict(mesh_nx=(256,) * 3, block_nx=(n,) * 3, pack_size=ps, **u),
                                                prob=2, par=BLAST)
    return c


def run(name, c, cycles, warmup):
    import torch
    import paper_2202_12309_b200 as P
    for k, v in c.get("env", {}).items():
        os.environ[k] = v
    try:
        m = P.Mesh(**c["kw"])
        m.set_problem(c["prob"], c["par"])
        m.step(warmup)
        torch.cuda.synchronize()
        l0 = m.launch_count()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = c["kw"]["block_nx"][0]
        amr = c["kw"].get("refinement") == 2
        zc = 0
        t0 = time.perf_counter()
        e0.record(s)
        if amr:  # the mesh changes every cycle: count the zones each cycle actually updates
            for _ in range(cycles):
                zc += m.num_blocks() * n ** 3
                m.step(1)
        else:
            m.step(cycles)
        e1.record(s)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ms = e0.elapsed_time(e1)
        nb = m.num_blocks()
        hist = m.history()
        if not amr:
            zc = nb * n ** 3 * cycles
        out = dict(config=name, blocks=nb, block=n, cycles=cycles, ms_per_cycle=ms / cycles,
                   wall_ms_per_cycle=wall * 1e3 / cycles, zone_cycles_per_s=zc / (ms * 1e-3),
                   launches_per_cycle=(m.launch_count() - l0) / cycles,
                   pack_size=c["kw"].get("pack_size", 0), mass_drift=float(abs(hist[-1, 2] - hist[0, 2]) / hist[0, 2]))
        m.close()
    finally:
        for k in c.get("env", {}):
            os.environ.pop(k, None)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    C = cases()
    names = [n for n in C if not a.only or any(n == o or n.startswith(o + "-") for o in a.only.split(","))]
    for n in names:
        try:
            print(json.dumps(run(n, C[n], a.cycles, a.warmup)), flush=True)
        except Exception as e:  # keep sweeping
            print(json.dumps(dict(config=n, error=str(e))), flush=True)


if __name__ == "__main__":
    main()
