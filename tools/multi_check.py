"""Multi-GPU parity check, launched with torchrun (one process per GPU, NCCL):

    torchrun --nproc-per-node N --master-addr 127.0.0.1 --master-port P tools/multi_check.py [--case blast] [--halo peer]

Every rank runs its Morton range; rank 0 gathers all blocks and compares them with (a) the CPU
oracle (1e-12, tests/parity.py) and (b) a single-GPU run of the same problem (bitwise)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CASES = {
    "blast": dict(kw=dict(mesh_nx=(64, 64, 64), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3),
                  problem=2, params=[10.0, 0.1, 0.15], cycles=10),
    "sod_walls": dict(kw=dict(mesh_nx=(128, 32, 32), block_nx=(16, 16, 16), gamma=1.4,
                              bc_inner=(1, 2, 0), bc_outer=(1, 2, 0)),
                      problem=1, params=[0.5], cycles=10),
    "wave64": dict(kw=dict(mesh_nx=(128, 64, 64), block_nx=(32, 32, 32)), problem=0,
                   params=[1e-6, 1, 1, 1], cycles=10),
    # static multilevel: coarse-fine faces (flux correction) and level-jump ghosts cross ranks
    "smr2": dict(kw=dict(mesh_nx=(32, 32, 32), block_nx=(8, 8, 8), xmin=(-.5,) * 3, xmax=(.5,) * 3, max_level=1,
                         refinement=1, regions=[(1, -0.15, 0.15, -0.15, 0.15, -0.15, 0.15)]),
                 problem=2, params=[10.0, 0.1, 0.12], cycles=10),
    "smr3_walls": dict(kw=dict(mesh_nx=(32, 16, 16), block_nx=(8, 8, 8), max_level=2, refinement=1, gamma=1.4,
                               regions=[(2, 0.45, 0.55, 0.2, 0.6, 0.3, 0.7)], bc_inner=(1, 1, 2), bc_outer=(1, 2, 1)),
                       problem=1, params=[0.5], cycles=10),
    # NEXT 3: WENO-Z with nghost 3 (generic high-order path) across GPUs
    "wenoz": dict(kw=dict(mesh_nx=(64, 32, 32), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3, recon=4,
                          nghost=3), problem=2, params=[10.0, 0.1, 0.15], cycles=8),
    # fewer blocks than ranks: some ranks own no block at all (empty partitions, A19/O2)
    "tiny": dict(kw=dict(mesh_nx=(64, 32, 32), block_nx=(32, 32, 32), xmin=(-.5,) * 3, xmax=(.5,) * 3),
                 problem=2, params=[10.0, 0.1, 0.2], cycles=6),
    # AMR: tagging gathered across ranks, remesh with block migration between GPUs
    "amr2": dict(kw=dict(mesh_nx=(32, 32, 32), block_nx=(8, 8, 8), xmin=(-.5,) * 3, xmax=(.5,) * 3, max_level=2,
                         refinement=2, refine_tol=0.1, derefine_tol=0.025, derefine_interval=2),
                 problem=2, params=[10.0, 0.1, 0.1], cycles=10),
    # AMR with 16^3 blocks: stage2's multilevel variant, the TMA tag pass, remesh + migration
    "amr16": dict(kw=dict(mesh_nx=(64, 64, 64), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3, max_level=2,
                          refinement=2, refine_tol=0.1, derefine_tol=0.025, derefine_interval=2),
                  problem=2, params=[10.0, 0.1, 0.1], cycles=8),
}


def run_case(P, case, halo, cycles, rank, world, local):
    import numpy as np
    import torch.distributed as dist
    C = dict(CASES[case])
    if cycles > 0:
        C["cycles"] = cycles
    transport = {"auto": P.HALO_AUTO, "nccl": P.HALO_NCCL, "peer": P.HALO_PEER}[halo]
    m = P.Mesh(device=local, rank=rank, nranks=world, halo_transport=transport, **C["kw"])
    m.set_problem(C["problem"], C["params"])
    m.step(C["cycles"])
    mine = {b["gid"]: m.get_state(b["gid"]) for b in m.blocks() if b["rank"] == rank}
    hist = m.history()
    tm = m.time()
    info = m.plan_info()
    objs = [None] * world
    dist.gather_object(mine, objs if rank == 0 else None, dst=0)
    ok = True
    if rank == 0:
        import oracle as O
        from parity import errors
        allb = {}
        for o in objs:
            allb.update(o)
        G = np.stack([allb[g] for g in sorted(allb)])
        orc = O.Mesh(**C["kw"])
        orc.set_problem(C["problem"], C["params"])
        orc.step(C["cycles"])
        Og = np.stack([orc.get_state(g) for g in range(orc.num_blocks())])
        e = errors(G, Og)
        single = P.Mesh(device=local, **C["kw"])
        single.set_problem(C["problem"], C["params"])
        single.step(C["cycles"])
        S = np.stack([single.get_state(g) for g in range(single.num_blocks())])
        single.close()
        bitwise = bool(S.shape == G.shape and np.array_equal(S, G))
        same_mesh = [(b["gid"], b["level"], b["lx"]) for b in orc.blocks()] == \
            [(b["gid"], b["level"], b["lx"]) for b in m.blocks()]
        to = orc.time()
        ho = orc.history()
        res = dict(case=case, world=world, parity=e, max_err=max(e.values()), bitwise_vs_1gpu=bitwise,
                   same_mesh=same_mesh, nblocks=len(allb),
                   t=tm, t_oracle=to, dt_rel=abs(tm[1] - to[1]) / to[1],
                   mass_rel=float(abs(hist[-1, 2] - ho[-1, 2]) / ho[-1, 2]),
                   send_doubles=info["send_doubles_to"], halo=halo, peer_halo=info["peer_halo"])
        ok = res["max_err"] <= 1e-12 and bitwise and same_mesh and res["dt_rel"] <= 1e-12 and tm[2] == to[2]
        ok = ok and (info["peer_halo"] == (halo == "peer") or halo == "auto")
        res["ok"] = ok
        print("MULTI_CHECK " + json.dumps(res), flush=True)
    m.close()
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="blast")
    ap.add_argument("--halo", default="auto", choices=["auto", "nccl", "peer"])
    ap.add_argument("--cases", default="",
                    help="comma-separated case:halo list run in this one process group (one torchrun start "
                         "for many cases); overrides --case / --halo")
    ap.add_argument("--cycles", type=int, default=0, help="override the case's cycle count (soak runs)")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    import paper_2202_12309_b200 as P
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    todo = [tuple(c.split(":")) for c in a.cases.split(",") if c] or [(a.case, a.halo)]
    ok = True
    for case, halo in todo:
        ok = run_case(P, case, halo, a.cycles, rank, world, local) and ok
        dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
