"""CPU tests of the C-ABI library (no GPU): it loads, exports every symbol include/ph.h declares,
and its host-side mesh (independent of the oracle's) matches the oracle bit for bit:
block list, Morton gids, rank assignment and canonical neighbour lists."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    from paper_2202_12309_b200 import _build
    _build.build()
    import paper_2202_12309_b200 as P
    return P


def test_library_exports_every_declared_symbol(P):
    hdr = open(os.path.join(ROOT, "include", "ph.h")).read()
    names = set(re.findall(r"^(?:ph_status|const char\*)\s+(ph_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 20
    L = P.lib()
    for n in sorted(names):
        assert hasattr(L, n), n
    assert set(P.ph.EXPORTS) == names


def test_oracle_header_and_product_header_share_nothing():
    prod = open(os.path.join(ROOT, "include", "ph.h")).read()
    assert "oracle" not in prod.lower().replace("oracle/", "")
    for f in os.listdir(os.path.join(ROOT, "paper_2202_12309_b200", "csrc")):
        src = open(os.path.join(ROOT, "paper_2202_12309_b200", "csrc", f)).read()
        assert "oracle.h" not in src and "orc_" not in src, f
    for f in ("ph.py", "__init__.py", "_build.py"):
        src = open(os.path.join(ROOT, "paper_2202_12309_b200", f)).read()
        assert "import oracle" not in src and "from oracle" not in src


def test_config_errors(P):
    with pytest.raises(P.PhError) as e:
        P.Mesh(host_only=True, mesh_nx=(30, 32, 32), block_nx=(16, 16, 16))
    assert e.value.code == 2
    with pytest.raises(P.PhError):
        P.Mesh(host_only=True, bc_inner=(0, 0, 1), bc_outer=(0, 0, 0))
    with pytest.raises(P.PhError):
        P.Mesh(host_only=True, nghost=4)
    with pytest.raises(P.PhError):
        P.Mesh(host_only=True, recon=P.WENOZ, nghost=2)
    with pytest.raises(P.PhError):
        P.Mesh(host_only=True, nghost=3, mesh_nx=(16,) * 3, block_nx=(8,) * 3, max_level=1, refinement=1,
               regions=[(1, 0, 0.5, 0, 0.5, 0, 0.5)])
    P.Mesh(host_only=True, recon=P.PPM, nghost=3)


def _compare_meshes(O, P, nranks=1, **kw):
    okw = dict(kw)
    o = O.Mesh(nranks=nranks, **okw)
    ob = o.blocks()
    for r in range(nranks):
        p = P.Mesh(host_only=True, rank=r, nranks=nranks, **kw)
        pb = p.blocks()
        assert len(ob) == len(pb)
        for a, b in zip(ob, pb):
            assert (a["gid"], a["level"], a["rank"], a["lx"]) == (b["gid"], b["level"], b["rank"], b["lx"])
            assert a["xmin"] == b["xmin"] and a["xmax"] == b["xmax"]
        for g in range(len(ob)):
            assert o.neighbors(g) == p.neighbors(g), g
    return len(ob)


def test_paper_mesh_matches_oracle(oracle_mod, P):
    n = _compare_meshes(oracle_mod, P, nranks=8, mesh_nx=(256,) * 3, block_nx=(32,) * 3, max_level=3,
                        refinement=1, regions=[(3, 0.3, 0.7, 0.3, 0.7, 0.3, 0.7)])
    assert n == 24816


@pytest.mark.parametrize("R,root", [(1, (4, 4, 4)), (2, (8, 4, 4)), (4, (8, 8, 4)), (8, (8, 8, 8))])
def test_weak_configs_match_oracle(oracle_mod, P, R, root):
    _compare_meshes(oracle_mod, P, nranks=R, mesh_nx=tuple(64 * r for r in root), block_nx=(64,) * 3,
                    xmin=(-0.5,) * 3, xmax=(-0.5 + root[0] / 4, -0.5 + root[1] / 4, -0.5 + root[2] / 4))


def test_random_multilevel_meshes_match_oracle(oracle_mod, P):
    rng = np.random.default_rng(20220224)
    for trial in range(25):
        root = tuple(int(x) for x in rng.integers(1, 4, size=3))
        L = int(rng.integers(1, 4))
        periodic = [bool(x) for x in rng.integers(0, 2, size=3)]
        regs = []
        for _ in range(int(rng.integers(1, 4))):
            r = [int(rng.integers(1, L + 1))]
            for d in range(3):
                a, b = sorted(rng.uniform(0, 1, 2))
                r += [a, b + 1e-3]
            regs.append(r)
        bc = tuple(0 if p else int(rng.integers(1, 3)) for p in periodic)
        _compare_meshes(oracle_mod, P, nranks=int(rng.integers(1, 5)), mesh_nx=tuple(8 * r for r in root),
                        block_nx=(8, 8, 8), max_level=L, refinement=1, regions=regs, bc_inner=bc, bc_outer=bc)


def test_exchange_plan_is_symmetric_across_ranks(P):
    """What rank s packs for rank d is exactly what d unpacks from s (sizes and order)."""
    for R in (2, 3, 4, 8):
        kw = dict(mesh_nx=(128, 64, 64), block_nx=(16, 16, 16), max_level=1, refinement=1,
                  regions=[(1, 0.2, 0.5, 0.3, 0.6, 0.1, 0.4)])
        infos = [P.Mesh(host_only=True, rank=r, nranks=R, **kw).plan_info() for r in range(R)]
        for s in range(R):
            for d in range(R):
                if s == d:
                    assert infos[s]["send_doubles_to"][d] == 0
                    continue
                assert infos[s]["send_doubles_to"][d] == infos[d]["recv_doubles_from"][s]
                assert infos[s]["send_hash_to"][d] == infos[d]["recv_hash_from"][s]
    # one rank: everything is local
    info = P.Mesh(host_only=True, mesh_nx=(64, 64, 64), block_nx=(16, 16, 16)).plan_info()
    assert info["n_send_tasks"] == 0 and info["n_recv_tasks"] == 0
    assert info["n_local_tasks"] == 64 * 26


def test_weak_8rank_plan_has_7_peers(P):
    """in the 8-GPU weak config every rank exchanges with all 7 peers."""
    for r in range(8):
        info = P.Mesh(host_only=True, rank=r, nranks=8, mesh_nx=(512,) * 3, block_nx=(64,) * 3).plan_info()
        peers = [p for p in range(8) if info["send_doubles_to"][p] > 0]
        assert len(peers) == 7


def test_direct_halo_cycle_plan(P):
    # uniform periodic single rank: the per-cycle exchange is empty (all faces read directly)
    info = P.Mesh(host_only=True, mesh_nx=(64, 64, 64), block_nx=(16, 16, 16)).plan_info()
    assert info["direct_halo"] and info["n_cyc_local_tasks"] == 0
    # multilevel: blocks without a coarser neighbour read their same-level local faces directly and
    # drop edge / corner ghosts; blocks with coarse staging keep every entry.  The per-cycle plan is
    # therefore a strict subset of the full one, and the direct halo can be switched off.
    ml = dict(mesh_nx=(64, 64, 64), block_nx=(16, 16, 16), max_level=1, refinement=1,
              regions=[(1, 0.1, 0.3, 0.1, 0.3, 0.1, 0.3)])
    info = P.Mesh(host_only=True, **ml).plan_info()
    assert info["direct_halo"] and 0 < info["n_cyc_local_tasks"] < info["n_local_tasks"]
    off = P.Mesh(host_only=True, direct_halo=False, **ml).plan_info()
    assert not off["direct_halo"] and off["n_cyc_local_tasks"] == off["n_local_tasks"] == info["n_local_tasks"]
    # multi-rank uniform, NCCL halo: the cycle plan keeps only remote faces, symmetric across ranks
    R = 4
    kw = dict(mesh_nx=(128, 64, 64), block_nx=(16, 16, 16), halo_transport=P.HALO_NCCL)
    infos = [P.Mesh(host_only=True, rank=r, nranks=R, **kw).plan_info() for r in range(R)]
    for s in range(R):
        for d in range(R):
            assert infos[s]["cyc_send_doubles_to"][d] == infos[d]["cyc_recv_doubles_from"][s]
            assert infos[s]["cyc_send_hash_to"][d] == infos[d]["cyc_recv_hash_from"][s]
            assert infos[s]["cyc_send_doubles_to"][d] <= infos[s]["send_doubles_to"][d]
    assert any(i["cyc_send_doubles_to"][d] > 0 for i in infos for d in range(R))
    assert all(i["n_cyc_local_tasks"] == 0 and not i["peer_halo"] for i in infos)


def test_peer_halo_plan(P):
    """Peer transport (uniform, N > 1): the per-cycle plan is the NCCL one -- what rank s puts into d's
    receive buffer is exactly what d unpacks from s -- and only the transport differs."""
    R = 4
    for bc in (P.PERIODIC, P.OUTFLOW):
        kw = dict(mesh_nx=(128, 64, 64), block_nx=(16, 16, 16), bc_inner=(bc,) * 3, bc_outer=(bc,) * 3)
        peer = [P.Mesh(host_only=True, rank=r, nranks=R, **kw).plan_info() for r in range(R)]
        nccl = [P.Mesh(host_only=True, rank=r, nranks=R, halo_transport=P.HALO_NCCL, **kw).plan_info()
                for r in range(R)]
        for i, j in zip(peer, nccl):
            assert i["peer_halo"] and i["direct_halo"] and not j["peer_halo"]
            for key in ("cyc_send_doubles_to", "cyc_recv_doubles_from", "cyc_send_hash_to", "cyc_recv_hash_from"):
                assert i[key] == j[key]
            assert sum(i["cyc_send_doubles_to"]) > 0
    # static multilevel and adaptive meshes are eligible (a remesh rebuilds the peer regions); not: one
    # rank, nghost 3, NCCL forced, no direct halo
    ml = dict(max_level=1, refinement=1, regions=[(1, 0.1, 0.3, 0.1, 0.3, 0.1, 0.3)])
    assert P.Mesh(host_only=True, rank=0, nranks=2, mesh_nx=(64,) * 3, block_nx=(16,) * 3, **ml).plan_info()["peer_halo"]
    amr = dict(max_level=1, refinement=P.REF_ADAPTIVE)
    assert P.Mesh(host_only=True, rank=0, nranks=2, mesh_nx=(64,) * 3, block_nx=(16,) * 3, **amr).plan_info()["peer_halo"]
    assert not P.Mesh(host_only=True, mesh_nx=(64,) * 3, block_nx=(16,) * 3).plan_info()["peer_halo"]
    for extra in (dict(nghost=3, recon=P.PPM), dict(direct_halo=False), dict(halo_transport=P.HALO_NCCL)):
        i = P.Mesh(host_only=True, rank=0, nranks=2, mesh_nx=(64,) * 3, block_nx=(16,) * 3, **extra).plan_info()
        assert not i["peer_halo"]
    # requiring it where it cannot apply is an error, as is an unknown transport
    with pytest.raises(P.PhError) as e:
        P.Mesh(host_only=True, rank=0, nranks=2, mesh_nx=(64,) * 3, block_nx=(16,) * 3, halo_transport=P.HALO_PEER,
               direct_halo=False)
    assert e.value.code == 8
    with pytest.raises(P.PhError):
        P.Mesh(host_only=True, mesh_nx=(64,) * 3, block_nx=(16,) * 3, halo_transport=7)
