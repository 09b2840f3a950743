"""The CPU-baseline plan of BASELINE.md §3 / SURVEY §8(d): the oracle (plain scalar C++, as it stands)
on BASELINE configs 1, 2a and 3 for 10 cycles, on 1 thread and on all host cores, with the CPU model.

    python tools/cpu_baseline.py [--cycles 10] [--out profiles/r02_cpu_baseline.json]

Run on the GPU box's host (gpurun); bench.py's cpu_baseline quotes the committed result beside its own
bounded sample.  Config 3 is timed including its AMR tag / remesh work, after the t = 0
pre-refinement (not timed)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CONFIGS = {
    "1": dict(kw=dict(mesh_nx=(32, 32, 32), block_nx=(32, 32, 32)), problem=0, params=[1e-6, 1, 1, 1],
              desc="linear wave, 32^3 mesh = 1 block of 32^3"),
    "2a": dict(kw=dict(mesh_nx=(256, 256, 256), block_nx=(64, 64, 64), xmin=(-.5,) * 3, xmax=(.5,) * 3),
               problem=2, params=[10.0, 0.1, 0.1], desc="blast, 256^3 mesh of 64^3 blocks (64 blocks)"),
    "3": dict(kw=dict(mesh_nx=(128, 128, 128), block_nx=(32, 32, 32), xmin=(-.5,) * 3, xmax=(.5,) * 3, max_level=3,
                      refinement=2, refine_tol=0.1, derefine_tol=0.025, derefine_interval=8),
              problem=2, params=[10.0, 0.1, 0.1], desc="blast AMR, 128^3 root of 32^3 blocks, 3 levels"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=10)
    ap.add_argument("--configs", default="1,2a,3")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_cpu_baseline.json"))
    a = ap.parse_args()
    import oracle as O
    from bench import cpu_model
    O.build()
    cores = len(os.sched_getaffinity(0))
    rows = []
    for name in a.configs.split(","):
        C = CONFIGS[name]
        for threads in (1, cores):
            m = O.Mesh(nthreads=threads, **C["kw"])
            m.set_problem(C["problem"], C["params"])
            n3 = 1
            for x in C["kw"]["block_nx"]:
                n3 *= x
            cells0 = m.num_blocks() * n3
            t0 = time.perf_counter()
            zc = 0
            for _ in range(a.cycles):  # count the cells of every cycle (the AMR mesh grows)
                zc += m.num_blocks() * n3
                m.step(1)
            dt = time.perf_counter() - t0
            row = dict(config=name, desc=C["desc"], threads=threads, cycles=a.cycles, blocks_start=cells0 // n3,
                       blocks_end=m.num_blocks(), zone_cycles=zc, seconds=dt, zone_cycles_per_s=zc / dt)
            print(json.dumps(row), flush=True)
            rows.append(row)
            m.close()
    res = {"cpu_model": cpu_model(), "cores": cores, "oracle": "oracle/oracle.cpp, g++ -O2 -ffp-contract=off, "
           "OpenMP across blocks", "rows": rows}
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
