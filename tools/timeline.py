"""Kernel timeline of a few multi-GPU cycles (the nsys substitute: this image has no nsys; torch.profiler
records every kernel, ours included, through CUPTI with its stream and timestamps).

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/timeline.py [--cycles 2] [--out profiles/r02_timeline_n4]

Rank 0 writes <out>.json (kernels: name, stream, start, duration, relative to the first kernel) and
<out>.md: per stream busy time, the time both streams run at once (boundary-first overlap, P:1274-1285:
the boundary blocks and their halo on stream B while the interior blocks run on stream I), and where
the halo kernels (put / pack / wait) sit relative to the interior stage kernels."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def intervals_union(iv):
    iv = sorted(iv)
    out = []
    for s, e in iv:
        if out and s <= out[-1][1]:
            out[-1][1] = max(out[-1][1], e)
        else:
            out.append([s, e])
    return out


def overlap(a, b):
    i = j = 0
    tot = 0.0
    while i < len(a) and j < len(b):
        s, e = max(a[i][0], b[j][0]), min(a[i][1], b[j][1])
        if e > s:
            tot += e - s
        if a[i][1] < b[j][1]:
            i += 1
        else:
            j += 1
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=2)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "timeline"))
    ap.add_argument("--config", default="2b", choices=["2b", "3"], help="3: the AMR blast on one GPU")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    from torch.profiler import ProfilerActivity, profile
    import paper_2202_12309_b200 as P
    from bench import BLAST, workload
    rank, world, local = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if a.config == "3":
        W = dict(mesh_nx=(128,) * 3, block_nx=(32,) * 3, max_level=3, refinement=2, refine_tol=0.1,
                 derefine_tol=0.025, derefine_interval=8, xmin=(-.5,) * 3, xmax=(.5,) * 3)
    else:
        W = workload("2b", world)
    m = P.Mesh(device=local, rank=rank, nranks=world, stream=torch.cuda.current_stream(), **W)
    m.set_problem(P.BLAST, BLAST)
    m.step(3)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        m.step(a.cycles)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if rank == 0:
        trace = a.out + "_trace.json"
        prof.export_chrome_trace(trace)
        ev = json.load(open(trace))
        ev = ev["traceEvents"] if isinstance(ev, dict) else ev
        ks = [e for e in ev if e.get("cat") == "kernel"]
        t0 = min(e["ts"] for e in ks)
        rows = [{"name": e["name"][:80], "stream": e.get("args", {}).get("stream"), "start_us": e["ts"] - t0,
                 "dur_us": e["dur"]} for e in sorted(ks, key=lambda e: e["ts"])]
        json.dump({"world": world, "cycles": a.cycles, "kernels": rows}, open(a.out + ".json", "w"), indent=0)
        os.remove(trace)
        streams = sorted({r["stream"] for r in rows}, key=lambda s: (s is None, s))
        busy = {s: intervals_union([(r["start_us"], r["start_us"] + r["dur_us"]) for r in rows if r["stream"] == s])
                for s in streams}
        span = max(r["start_us"] + r["dur_us"] for r in rows)
        stage = [r for r in rows if "stage" in r["name"]]
        # the stream that runs the most stage time is the interior stream I
        by = {s: sum(r["dur_us"] for r in stage if r["stream"] == s) for s in streams}
        si = max(by, key=by.get)
        others = [s for s in streams if s != si]
        halo = [r for r in rows if any(k in r["name"] for k in ("xfill", "peer_wait", "peer_signal", "nccl", "Nccl"))]
        with open(a.out + ".md", "w") as f:
            f.write(f"# kernel timeline, {world} GPUs, rank 0, {a.cycles} cycles (torch.profiler / CUPTI)\n\n")
            f.write(f"span {span:.0f} us; kernels {len(rows)}\n\n| stream | kernels | busy us | overlap with interior stream us |\n|---|---|---|---|\n")
            for s in streams:
                n = sum(1 for r in rows if r["stream"] == s)
                b = sum(e - s_ for s_, e in busy[s])
                ov = overlap(busy[s], busy[si]) if s != si else 0.0
                f.write(f"| {s}{' (interior I)' if s == si else ''} | {n} | {b:.0f} | {ov:.0f} |\n")
            f.write("\n| kernel | stream | start us | dur us |\n|---|---|---|---|\n")
            for r in rows[:80]:
                f.write(f"| {r['name'][:60]} | {r['stream']} | {r['start_us']:.0f} | {r['dur_us']:.0f} |\n")
            tot = {}
            for r in rows:
                k = r["name"][:60]
                tot[k] = tot.get(k, [0, 0.0])
                tot[k][0] += 1
                tot[k][1] += r["dur_us"]
            f.write("\n| kernel (all launches) | launches | total us |\n|---|---|---|\n")
            for k, (n_, t_) in sorted(tot.items(), key=lambda x: -x[1][1]):
                f.write(f"| {k} | {n_} | {t_:.0f} |\n")
            busy_all = intervals_union([(r["start_us"], r["start_us"] + r["dur_us"]) for r in rows])
            f.write(f"\nGPU busy {sum(e - s_ for s_, e in busy_all):.0f} us of {span:.0f} us span (idle gaps = host work / launch latency)\n")
            hin = sum(r["dur_us"] for r in halo)
            # overlap = halo time during which a stage kernel runs on another stream (0 on one stream)
            hov = 0.0
            for hs in {r["stream"] for r in halo}:
                h_iv = intervals_union([(r["start_us"], r["start_us"] + r["dur_us"]) for r in halo if r["stream"] == hs])
                st_iv = intervals_union([(r["start_us"], r["start_us"] + r["dur_us"]) for r in stage if r["stream"] != hs])
                hov += overlap(h_iv, st_iv)
            f.write(f"\nhalo kernels (pack / put / signal / wait / NCCL): {hin:.0f} us, of which {hov:.0f} us "
                    f"run while a stage kernel computes on another stream\n")
        print(open(a.out + ".md").read()[:1500])
    m.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
