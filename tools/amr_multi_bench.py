"""Config 3 (AMR blast, 128³ root, 32³ blocks, 3 levels) on N GPUs: ms per cycle with the peer-memory
halo (rebuilt at every remesh) vs NCCL, CUDA events around 10 cycles, max over ranks.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port P tools/amr_multi_bench.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import paper_2202_12309_b200 as P
    rank, world, local = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    kw = dict(mesh_nx=(128,) * 3, block_nx=(32,) * 3, max_level=3, refinement=P.REF_ADAPTIVE, refine_tol=0.1,
              derefine_tol=0.025, derefine_interval=8, xmin=(-.5,) * 3, xmax=(.5,) * 3)
    out = {}
    for halo, tr in (("peer", P.HALO_PEER), ("nccl", P.HALO_NCCL)):
        m = P.Mesh(device=local, rank=rank, nranks=world, halo_transport=tr, stream=torch.cuda.current_stream(), **kw)
        m.set_problem(P.BLAST, [10.0, 0.1, 0.1])
        m.step(3)
        torch.cuda.synchronize()
        dist.barrier()
        nb0 = m.num_blocks()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m.step(10)
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / 10], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        zc = 0
        for b in m.blocks():
            zc += 32 ** 3
        out[halo] = dict(ms_per_cycle=ms.item(), blocks_start=nb0, blocks_end=m.num_blocks(),
                         zone_cycles_per_s=zc / (ms.item() * 1e-3), peer_halo=m.plan_info()["peer_halo"])
        m.close()
        dist.barrier()
    if rank == 0:
        print(json.dumps(dict(world=world, **out)))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
