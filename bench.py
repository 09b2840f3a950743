#!/usr/bin/env python
"""Benchmark of the B200 Parthenon-hydro hot path: zone-cycles/s (BASELINE.json metric).

One step = one full RK2 cycle of the hot path (stage 1, ghost exchange, stage 2, ghost
exchange, CFL dt reduction + conserved totals) over all blocks of every GPU.

Default workload (N=1): BASELINE configs[1] in reading 2b (SURVEY finding 1): 3D blast wave,
512^3 mesh of 64^3 blocks (512 blocks), all blocks in one launch, fp64.  For N>1 the per-GPU
work is fixed (weak scaling): the global mesh grows along the Morton axes (1024x512x512, ...),
so every GPU owns a contiguous Morton range of 512 blocks.  --config 4 selects BASELINE
configs[3] (256^3 cells per GPU).

    python bench.py --gpus N --steps K --warmup W [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PER_GPU_ROOT = {"2b": (8, 8, 8), "4": (4, 4, 4)}
SCALE_AXES = [(1, 1, 1), (2, 1, 1), (2, 2, 1), (2, 2, 2), (4, 2, 2), (4, 4, 2), (4, 4, 4), (8, 4, 4)]


def workload(cfg, ngpu, n=64, strong=False):
    root = PER_GPU_ROOT[cfg]
    k = {1: 0, 2: 1, 4: 2, 8: 3}.get(ngpu)
    if k is None:
        raise SystemExit(f"--gpus {ngpu}: use 1, 2, 4 or 8")
    ax = SCALE_AXES[0 if strong else k]  # strong scaling: the 1-GPU mesh on every N
    groot = tuple(root[d] * ax[d] for d in range(3))
    mesh = tuple(n * r for r in groot)
    # unit cell width in every direction: domain extents proportional to the mesh
    L = tuple(m / (n * root[0]) for m in mesh)
    xmin = tuple(-0.5 * l for l in L)
    xmax = tuple(0.5 * l for l in L)
    return dict(mesh_nx=mesh, block_nx=(n, n, n), xmin=xmin, xmax=xmax)


BLAST = [10.0, 0.1, 0.1]  # p_in, p_out, radius (A21), centred in the global domain


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler during the timed region (the recipe's clocks line)."""

    def __init__(self, idx):
        self.idx = idx
        self.proc = None
        self.lines = []

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0, set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for name, val in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------------------ oracle legs
def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(cfg_name, steps, warmup, threads, mesh_n=256):
    """The CPU oracle (as it stands) on a bounded sample of the workload: the same 64^3 blocks,
    method and blast problem on a 256^3 periodic mesh (BASELINE configs[1] as written = reading 2a:
    64 blocks, at least one per core); one oracle cycle per step."""
    import oracle
    oracle.build()
    h = 0.5 * mesh_n / 256
    kw = dict(mesh_nx=(mesh_n,) * 3, block_nx=(64, 64, 64), xmin=(-h,) * 3, xmax=(h,) * 3, nthreads=threads)
    m = oracle.Mesh(**kw)
    m.set_problem(oracle.BLAST, BLAST)
    cells = mesh_n ** 3
    for _ in range(warmup):
        m.step(1)
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        m.step(1)
        ts.append(time.perf_counter() - t0)
    total = sum(ts)
    nb = (mesh_n // 64) ** 3
    return cells * steps / total, total / steps, (f"blast, {mesh_n}^3 periodic mesh of 64^3 blocks ({nb} blocks), "
                                                   f"{steps} oracle cycle(s), {threads} OpenMP thread(s)")


def cpu_baseline_block(steps):
    """cpu_baseline object: all host cores on the 2a sample, one thread on one 64^3 block, the CPU model,
    and the full BASELINE.md §3 plan as last measured on a GPU box (tools/cpu_baseline.py)."""
    threads = len(os.sched_getaffinity(0))
    zcs, sec, sample = oracle_sample("2a", steps, 0, threads)
    z1, s1, sample1 = oracle_sample("1blk", 1, 0, 1, mesh_n=64)
    out = {"value": zcs, "unit": "zone-cycles/s", "cores": threads, "kind": "oracle", "sample": sample,
           "cpu_model": cpu_model(),
           "single_thread": {"value": z1, "unit": "zone-cycles/s", "cores": 1, "sample": sample1}}
    fp = os.path.join(ROOT, "profiles", "r02_cpu_baseline.json")
    if os.path.exists(fp):
        try:
            out["full_plan"] = {"source": "profiles/r02_cpu_baseline.json (tools/cpu_baseline.py, not this run)",
                                "rows": json.load(open(fp)).get("rows")}
        except Exception:
            pass
    return out


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = len(os.sched_getaffinity(0))
    zcs, sec, sample = oracle_sample(args.config, args.steps, args.warmup, threads)
    line = {
        "impl": "reference", "metric": "zone-cycles/s", "value": zcs, "unit": "zone-cycles/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"oracle sample of {args.config}", "sample": sample},
        "cpu_baseline": {"value": zcs, "unit": "zone-cycles/s", "cores": threads, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": zcs, "unit": "zone-cycles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ GPU leg
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2202_12309_b200 as P

    rank, world, local = dist_env()
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("launch with torchrun --nproc-per-node N for --gpus N > 1")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    W = workload(args.config, world, strong=args.scaling == "strong")
    transport = {"auto": P.HALO_AUTO, "nccl": P.HALO_NCCL, "peer": P.HALO_PEER}[args.halo]
    mesh = P.Mesh(device=local, rank=rank, nranks=world, stream=stream, halo_transport=transport, **W)
    halo = "local direct halo" if world == 1 else (
        "peer memory: the pack kernel stores boundary faces into the peer's receive buffer over NVLink "
        "(CUDA IPC), release / acquire flags" if mesh.plan_info()["peer_halo"]
        else "NCCL send/recv of remote faces")
    nglob = mesh.num_blocks()
    n = W["block_nx"][0]
    cells = nglob * n ** 3
    mesh.set_problem(P.BLAST, BLAST)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        mesh.step(1)
    barrier()
    l0 = mesh.launch_count()
    mesh.kernel_timing(True)
    clk = Clocks(local)
    clk.start()
    barrier()
    # an event at every cycle boundary (the paper quotes the median of several tens of
    # cycles): value stays total cells x K / total time, the median is reported beside it
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    evs[0].record(stream)
    for i in range(args.steps):
        mesh.step(1)
        evs[i + 1].record(stream)
    barrier()
    clocks = clk.stop()
    ms = evs[0].elapsed_time(evs[-1])
    per_cycle = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    med = statistics.median(per_cycle)
    stage_ms, stage_n, exch_ms, exch_n = mesh.kernel_timing(False)
    launches = mesh.launch_count() - l0
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = cells * args.steps / (ms_max * 1e-3)
    tm = torch.tensor([med], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    med_max = float(tm.item())

    # correctness guard: the run must still be physical and conserve mass
    hist = mesh.history()
    t0 = hist[0, 2] if len(hist) else 0.0
    mass_drift = abs(hist[-1, 2] - t0) / t0 if len(hist) else 0.0

    # ---- end-to-end through the public host-buffer call (H2D + cycle + D2H every step).  Every step is
    # one problem: its state comes from pinned host memory and goes back to it.  Problems alternate
    # between two meshes on two streams (ph_step_host_async / ph_sync), so one problem's device->host
    # copy overlaps the next one's host->device copy (PCIe is full duplex).
    nloc = mesh.num_local()
    e2e = None
    if not args.no_e2e:
        hin = torch.empty((nloc, 5, n, n, n), dtype=torch.float64).pin_memory()
        outs = [torch.empty_like(hin).pin_memory() for _ in range(2)]
        # initial state from the device (rank-local gather)
        gids = [b["gid"] for b in mesh.blocks() if b["rank"] == rank]
        for i, g in enumerate(gids):
            hin[i].copy_(torch.from_numpy(mesh.get_state(g)))
        mesh2 = P.Mesh(device=local, rank=rank, nranks=world, stream=torch.cuda.Stream(), halo_transport=transport, **W)
        meshes = [mesh, mesh2]
        e2e_steps = max(2, args.e2e_steps)
        for M, o in zip(meshes, outs):
            M.step_host(hin, o, 1)  # warm-up
        barrier()
        t_0 = time.perf_counter()
        for s in range(e2e_steps):
            M = meshes[s % 2]
            if s >= 2:
                M.sync()  # its previous problem is done (and its output buffer free)
            M.step_host_async(hin, outs[s % 2], 1)
        for M in meshes:
            M.sync()
        dt_e2e = time.perf_counter() - t_0
        tt = torch.tensor([dt_e2e], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        nbytes = hin.numel() * 8
        assert torch.equal(outs[0], outs[1])  # the same problem on both meshes gives the same answer
        e2e = {"value": cells * e2e_steps / float(tt.item()), "unit": "zone-cycles/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "note": "each step: H2D of the rank's whole state, refresh + 1 cycle, D2H of the state "
                       "(ph_step_host_async on two meshes / streams, %d steps)" % e2e_steps}
        mesh2.close()

    # per-rank stage-kernel time: a slow GPU paces every rank through the halo / dt dependencies
    stage_ranks = [stage_ms / max(stage_n, 1)]
    if world > 1:
        tl = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(world)]
        dist.all_gather(tl, torch.tensor([stage_ms / max(stage_n, 1)], dtype=torch.float64, device="cuda"))
        stage_ranks = [float(x.item()) for x in tl]

    # ---- roofline of the dominant kernel (the fused stage kernel)
    peak, peak_kind = measured_peaks()
    r = ((n + 4) / n) ** 3
    nloc_cells = nloc * n ** 3
    # algorithmic bytes per stage launch: read U with halo (r*40 B/cell), write 40 B/cell,
    # stage 2 also reads U^n at the cell (40 B/cell): averaged over the two stages
    # per launch: the timed cycles' total algorithmic bytes over the stage launches (N > 1 splits each
    # stage into a boundary and an interior launch; N = 1: one launch of all local blocks)
    stage_bytes = nloc_cells * (r * 40.0 + 60.0) * 2 * args.steps / max(stage_n, 1)
    stage_avg_ms = stage_ms / max(stage_n, 1)
    achieved = stage_bytes / (stage_avg_ms * 1e-3) / 1e9 if stage_n else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "stage_kernel_traffic.json")
    if os.path.exists(tp):
        try:
            d = json.load(open(tp))
            if d.get("workload") == args.config and d.get("n") == n:
                traffic = d.get("bytes_per_launch")
        except Exception:
            traffic = None
    b_ghost = (6 * r - 1) * 40.0
    size = "512^3" if args.config == "2b" else "256^3"
    base = (f"(BASELINE configs[{1 if args.config == '2b' else 3}]"
            f"{', reading 2b' if args.config == '2b' else ''}), global mesh {W['mesh_nx']}, "
            f"{nglob} blocks, all local blocks per launch, PLM-minmod + HLLE + RK2, CFL 0.3")
    if args.scaling == "strong":
        workload_desc = f"blast 3D, fixed {size} global mesh in 64^3 blocks split over {world} GPU(s), strong scaling " + base
    else:
        workload_desc = f"blast 3D, {size} cells per GPU in 64^3 blocks " + base
    # co-limiter (SURVEY §8(d) "report both"): the fp64 pipe.  Instructions per cell-stage from the
    # committed ncu capture of the current stage kernel (profiles/stage_kernel_counts.json); peak =
    # the measured fp64 lanes / clock / SM of profiles/r02_ubench_fp64.jsonl x 148 SMs x the median SM
    # clock of this run.
    fp64 = None
    pc = os.path.join(ROOT, "profiles", "stage_kernel_counts.json")
    pu = os.path.join(ROOT, "profiles", "r02_ubench_fp64.jsonl")
    if os.path.exists(pc) and os.path.exists(pu) and stage_n:
        try:
            cnt = json.load(open(pc))
            per_cell = float(cnt["fp64_inst_per_cell_stage"])
            rows = []
            for l in open(pu):
                try:
                    rows.append(json.loads(l))
                except ValueError:  # a non-finite entry (the optimised-away dsetp probe)
                    continue
            lanes = max(r["lane_ops_per_clk_per_sm"] for r in rows if r.get("op") in ("dfma", "dadd", "dmul"))
            mhz = (clocks or {}).get("sm_mhz") or 1965.0
            ach = per_cell * nloc_cells * 2 * args.steps / (stage_ms * 1e-3)  # all timed stage launches
            fpk = 148 * lanes * mhz * 1e6
            fp64 = {"bound": "alu", "achieved": ach, "peak": fpk, "unit": "fp64-pipe thread instr/s",
                    "frac": ach / fpk, "inst_per_cell_stage": per_cell,
                    "inst_total_per_cell_stage": cnt.get("thread_inst_per_cell_stage"),
                    "source": f"inst count: {cnt.get('source')}; peak: 148 SM x {lanes:.1f} lanes/clk "
                              f"(measured DADD/DMUL/DFMA, profiles/r02_ubench_fp64.jsonl) x {mhz:.0f} MHz"}
        except Exception:
            fp64 = None
    cyc_bytes = nloc_cells * (2 * r * 40.0 + 120.0)  # both stages, algorithmic (B_min), per GPU
    per_gpu = {"bytes_per_cycle": cyc_bytes, "ms_per_cycle": ms_max / args.steps,
               "achieved": cyc_bytes / (ms_max / args.steps * 1e-3) / 1e9,
               "frac": cyc_bytes / (ms_max / args.steps * 1e-3) / 1e9 / peak}
    line = {
        "metric": "zone-cycles/s", "value": value, "unit": "zone-cycles/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": workload_desc,
                   "global_blocks": nglob, "block": n, "nghost": 2,
                   "l2": "inputs larger than L2 (state %.1f GB per GPU vs 126 MB L2)" % (2 * nloc * 5 * (n + 4) ** 3 * 8 / 1e9),
                   "parallelism": f"morton-partition dp{world}", "halo": halo},
        "median": {"ms_per_step": med_max, "value": cells / (med_max * 1e-3),
                   "note": "median of per-cycle CUDA events (P:1005-1007), max over ranks"},
        "roofline": {"bound": "hbm", "achieved": achieved if world == 1 else per_gpu["achieved"], "peak": peak,
                     "unit": "GB/s",
                     "frac": ((achieved if world == 1 else per_gpu["achieved"]) / peak) if achieved else None,
                     "traffic": traffic,
                     "definition": ("algorithmic bytes per stage launch / mean launch time (CUDA events)" if world == 1
                                    else "per GPU: algorithmic bytes of both stages per cycle / cycle time "
                                         "(each stage is a boundary and an interior launch running concurrently)"),
                     "per_launch": {"achieved": achieved, "frac": (achieved / peak) if achieved else None},
                     "per_gpu_cycle": per_gpu,
                     "kernel": "stage kernel (stage2.cu: fused cons->prim, PLM, HLLE x/y/z, divergence, RK combine)",
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
                     "algorithmic_bytes_per_launch": stage_bytes,
                     "stage_ms_avg": stage_avg_ms, "stage_share_of_step": stage_ms / ms if ms else None,
                     "stage_ms_avg_per_rank": stage_ranks,
                     "exchange_ms_per_step": exch_ms / args.steps,
                     "cycle_hbm_frac_B_ghost": value / world * b_ghost / (peak * 1e9),
                     "B_ghost_bytes_per_zone_cycle": b_ghost, "fp64_pipe": fp64},
        "gpu_launches": launches,
        "clocks": clocks,
        "e2e": e2e,
        "mass_drift": mass_drift,
    }
    # ---- CPU baseline: the oracle on the host cores, rank 0 at N=1 only
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_block(args.cpu_steps)
    if rank == 0:
        print(json.dumps(line), flush=True)
    mesh.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="2b", choices=["2b", "4"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: fixed work per GPU (default); strong: the 1-GPU mesh split over N GPUs")
    ap.add_argument("--halo", default="auto", choices=["auto", "nccl", "peer"],
                    help="multi-GPU halo transport (auto: peer memory when every rank can map its peers)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=12)
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: W >= 3 warm-up steps required by the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
