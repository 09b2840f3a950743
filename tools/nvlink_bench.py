"""NVLink microbenchmarks of SURVEY §8(d) (once per box): per-peer copy bandwidth, all-peer
concurrent bandwidth, and the latency of the small collectives the cycle uses.

Single process (all visible GPUs):
    python tools/nvlink_bench.py --copy            # GPU0 -> GPUj peer copies, one at a time and all at once
Under torchrun (one process per GPU, NCCL):
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/nvlink_bench.py --coll
        # all_gather of 6 fp64 per rank (the dt / totals exchange) and all_reduce of 1 fp64 (8 B), us/op

Prints one JSON object per measurement (rank 0)."""
import argparse
import json
import os
import time


def copy_bench(mb):
    import torch
    n = torch.cuda.device_count()
    out = []
    nbytes = mb << 20
    src = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda:0").fill_(1.0)
    dsts = {j: torch.empty_like(src, device=f"cuda:{j}") for j in range(1, n)}
    for j, d in dsts.items():
        for _ in range(3):
            d.copy_(src, non_blocking=True)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(j)
        reps = 10
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(0):
            s0.record()
            for _ in range(reps):
                d.copy_(src, non_blocking=True)
            s1.record()
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(j)
        ms = s0.elapsed_time(s1) / reps
        out.append({"bench": "peer_copy", "src": 0, "dst": j, "bytes": nbytes, "ms": ms,
                    "GBps": nbytes / (ms * 1e-3) / 1e9})
    if len(dsts) > 1:  # GPU0 -> every peer at once (one stream per peer)
        streams = {j: torch.cuda.Stream(device=0) for j in dsts}
        torch.cuda.synchronize(0)
        t0 = time.perf_counter()
        reps = 10
        for _ in range(reps):
            for j, d in dsts.items():
                with torch.cuda.stream(streams[j]):
                    d.copy_(src, non_blocking=True)
        for j in dsts:
            torch.cuda.synchronize(j)
        torch.cuda.synchronize(0)
        dt = (time.perf_counter() - t0) / reps
        out.append({"bench": "peer_copy_all", "src": 0, "dst": list(dsts), "bytes_per_peer": nbytes,
                    "ms": dt * 1e3, "GBps_aggregate": nbytes * len(dsts) / dt / 1e9})
    return out


def coll_bench(iters):
    import torch
    import torch.distributed as dist
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    out = []
    for name, numel in (("all_gather_6xf64", 6), ("all_reduce_1xf64", 1)):
        x = torch.ones(numel, dtype=torch.float64, device="cuda")
        outs = [torch.empty_like(x) for _ in range(world)]
        def op():
            if name.startswith("all_gather"):
                dist.all_gather(outs, x)
            else:
                dist.all_reduce(x, op=dist.ReduceOp.MIN)
        for _ in range(20):
            op()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            op()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / iters
        t = torch.tensor([us], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out.append({"bench": name, "world": world, "bytes_per_rank": numel * 8, "us_per_op_max_rank": float(t.item())})
    dist.destroy_process_group()
    return out if rank == 0 else []


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--copy", action="store_true")
    ap.add_argument("--coll", action="store_true")
    ap.add_argument("--mb", type=int, default=256)
    ap.add_argument("--iters", type=int, default=2000)
    a = ap.parse_args()
    res = []
    if a.copy:
        res += copy_bench(a.mb)
    if a.coll:
        res += coll_bench(a.iters)
    for r in res:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
