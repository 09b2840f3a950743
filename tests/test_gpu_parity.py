"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tolerance: 1e-12 per cell with the floor of parity.py (north_star).
Integer outputs (block lists, ranks, neighbour lists) are compared bit-exactly elsewhere
(tests/test_lib_host.py); the exchange without arithmetic reordering is compared bitwise here.
"""
import numpy as np
import pytest

from parity import assert_parity, errors, gather

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    from paper_2202_12309_b200 import _build
    _build.build()
    import paper_2202_12309_b200 as P
    return P


def _pair(O, P, **kw):
    return O.Mesh(**kw), P.Mesh(**kw)


def _run_both(O, P, problem, params, cycles, tlim=0.0, **kw):
    o, g = _pair(O, P, **kw)
    o.set_problem(problem, params)
    g.set_problem(problem, params)
    # t = 0: both sides generate the same initial state and dt
    e0 = errors(gather(g), gather(o))
    assert max(e0.values()) <= 1e-15, e0
    assert abs(g.time()[1] - o.time()[1]) <= 1e-13 * o.time()[1]
    o.step(cycles, tlim)
    g.step(cycles, tlim)
    return o, g


def _check_run(o, g, tol=1e-12):
    e = assert_parity(gather(g), gather(o), tol)
    to, tg = o.time(), g.time()
    assert to[2] == tg[2]
    assert abs(tg[0] - to[0]) <= 1e-12 * max(to[0], 1e-300)
    assert abs(tg[1] - to[1]) <= 1e-12 * to[1]
    ho, hg = o.history(), g.history()
    assert ho.shape == hg.shape
    np.testing.assert_allclose(hg[:, :2], ho[:, :2], rtol=1e-12)
    np.testing.assert_allclose(hg[:, [2, 6]], ho[:, [2, 6]], rtol=1e-12)
    mom_scale = np.abs(gather(o)[:, 1:4]).sum() * 1e-12 + 1e-300
    assert np.all(np.abs(hg[:, 3:6] - ho[:, 3:6]) <= max(mom_scale, 1e-12 * np.abs(ho[:, 2]).max()))
    return e


def test_config1_linear_wave_single_block(oracle_mod, P):
    """BASELINE config 1: 3D linear wave, 32^3 mesh as one 32^3 block, 10 cycles."""
    o, g = _run_both(oracle_mod, P, P.LINEAR_WAVE, [1e-6, 1, 1, 1], 10,
                     mesh_nx=(32, 32, 32), block_nx=(32, 32, 32))
    _check_run(o, g)


def test_blast_many_blocks(oracle_mod, P):
    o, g = _run_both(oracle_mod, P, P.BLAST, [10.0, 0.1, 0.15], 10,
                     mesh_nx=(64, 64, 64), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3)
    _check_run(o, g)


def test_blast_ragged_tiles(oracle_mod, P):
    """block extents that are not multiples of the 32x8 tile: ragged tiles in x and y"""
    o, g = _run_both(oracle_mod, P, P.BLAST, [10.0, 0.1, 0.2], 10,
                     mesh_nx=(72, 36, 40), block_nx=(36, 12, 20), xmin=(-.5,) * 3, xmax=(.5,) * 3)
    _check_run(o, g)


def test_sod_thin_outflow(oracle_mod, P):
    kw = dict(mesh_nx=(256, 4, 4), block_nx=(64, 4, 4), gamma=1.4,
              bc_inner=(P.OUTFLOW, 0, 0), bc_outer=(P.OUTFLOW, 0, 0))
    o, g = _run_both(oracle_mod, P, P.SOD, [0.5], 100000, tlim=0.2, **kw)
    assert abs(g.time()[0] - 0.2) < 1e-15
    _check_run(o, g)


def test_blast_reflecting_walls(oracle_mod, P):
    kw = dict(mesh_nx=(32, 32, 32), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3,
              bc_inner=(P.REFLECT, P.OUTFLOW, P.REFLECT), bc_outer=(P.REFLECT, P.REFLECT, P.OUTFLOW))
    o, g = _run_both(oracle_mod, P, P.BLAST, [10.0, 0.1, 0.2, 0.1, -0.05, 0.0], 10, **kw)
    _check_run(o, g)


@pytest.mark.parametrize("recon,integ", [(1, 0), (2, 0), (0, 1)])
def test_limiters_and_vl2(oracle_mod, P, recon, integ):
    o, g = _run_both(oracle_mod, P, P.BLAST, [10.0, 0.1, 0.2], 8, recon=recon, integrator=integ,
                     mesh_nx=(32, 32, 32), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3)
    _check_run(o, g)


@pytest.mark.parametrize("integ", [0, 1])
def test_full_tile_stage2_base(oracle_mod, P, integ):
    """32^3 blocks take the full-tile path where stage 1 also writes the stage-2 base H = a0 U^n + b1 U^1
    (RK2: 1/2, 1/2; VL2: 1, 0) and stage 2 reads H instead of U^n and U^1 at the cell"""
    o, g = _run_both(oracle_mod, P, P.BLAST, [10.0, 0.1, 0.2, 0.1, -0.05, 0.0], 8, integrator=integ,
                     mesh_nx=(64, 64, 32), block_nx=(32, 32, 32), xmin=(-.5,) * 3, xmax=(.5,) * 3,
                     bc_inner=(P.REFLECT, P.PERIODIC, P.OUTFLOW), bc_outer=(P.REFLECT, P.PERIODIC, P.OUTFLOW))
    _check_run(o, g)


@pytest.mark.parametrize("case", ["blast", "sod_walls", "two_level"])
def test_einfeldt_wave_speeds(oracle_mod, P, case):
    """HLLE with Einfeldt (Roe-averaged) wave speeds (A4 variant, ph_config.wavespeed) vs the oracle"""
    u = dict(xmin=(-.5,) * 3, xmax=(.5,) * 3, wavespeed=P.EINFELDT)
    if case == "blast":
        o, g = _run_both(oracle_mod, P, P.BLAST, [10.0, 0.1, 0.2], 8, mesh_nx=(64, 64, 32), block_nx=(32, 32, 32), **u)
    elif case == "sod_walls":
        o, g = _run_both(oracle_mod, P, P.SOD, [0.5], 10, mesh_nx=(128, 16, 16), block_nx=(32, 16, 16), gamma=1.4,
                         wavespeed=P.EINFELDT, bc_inner=(P.OUTFLOW, P.REFLECT, 0), bc_outer=(P.REFLECT, P.OUTFLOW, 0))
    else:
        o, g = _run_both(oracle_mod, P, P.BLAST, [10.0, 0.1, 0.12], 10, mesh_nx=(32, 32, 32), block_nx=(8, 8, 8),
                         max_level=1, refinement=P.REF_STATIC, regions=[(1, -0.15, 0.15, -0.15, 0.15, -0.15, 0.15)], **u)
    _check_run(o, g)
    with pytest.raises(P.PhError):  # PPM / WENO-Z keep Davis speeds
        P.Mesh(mesh_nx=(32,) * 3, block_nx=(16,) * 3, nghost=3, recon=P.PPM, wavespeed=P.EINFELDT)


def test_static_two_level_blast_with_flux_correction(oracle_mod, P):
    kw = dict(mesh_nx=(32, 32, 32), block_nx=(8, 8, 8), xmin=(-.5,) * 3, xmax=(.5,) * 3, max_level=1,
              refinement=P.REF_STATIC, regions=[(1, -0.15, 0.15, -0.15, 0.15, -0.15, 0.15)])
    o, g = _run_both(oracle_mod, P, P.BLAST, [10.0, 0.1, 0.12], 10, **kw)
    _check_run(o, g)
    t0 = g.history()[0, 2:]
    t1 = g.totals()
    assert abs(t1[0] - t0[0]) <= 1e-12 * t0[0] and abs(t1[4] - t0[4]) <= 1e-12 * t0[4]


def test_static_multilevel_32cube_blocks_next1_path(oracle_mod, P):
    """The NEXT 1 (paper mesh) code path at a size the oracle finishes in seconds: exactly tiling 32^3
    blocks on a static 3-level mesh take the full-tile multilevel stage kernel with the fused dt /
    totals reduction and rfx_reduce_kernel (the corrected face layers reduced after the reflux)."""
    kw = dict(mesh_nx=(128, 128, 128), block_nx=(32, 32, 32), xmin=(-.5,) * 3, xmax=(.5,) * 3, max_level=2,
              refinement=P.REF_STATIC, regions=[(2, -0.12, 0.12, -0.12, 0.12, -0.12, 0.12)])
    o, g = _run_both(oracle_mod, P, P.BLAST, [10.0, 0.1, 0.1], 5, **kw)
    levels = [b["level"] for b in g.blocks()]
    assert set(levels) == {0, 1, 2}, sorted(set(levels))
    _check_run(o, g)
    t0 = g.history()[0, 2:]
    t1 = g.totals()
    assert abs(t1[0] - t0[0]) <= 1e-12 * t0[0] and abs(t1[4] - t0[4]) <= 1e-12 * t0[4]


def test_three_level_outflow_sod_like(oracle_mod, P):
    kw = dict(mesh_nx=(32, 16, 16), block_nx=(8, 8, 8), max_level=2, refinement=P.REF_STATIC, gamma=1.4,
              regions=[(2, 0.45, 0.55, 0.2, 0.6, 0.3, 0.7)], bc_inner=(1, 1, 2), bc_outer=(1, 2, 1))
    o, g = _run_both(oracle_mod, P, P.SOD, [0.5], 10, **kw)
    _check_run(o, g)


@pytest.mark.parametrize("multilevel", [False, True])
def test_exchange_bitwise(oracle_mod, P, multilevel):
    """restriction, prolongation, BCs and copies reproduce the oracle bit for bit"""
    kw = dict(mesh_nx=(32, 32, 24), block_nx=(8, 8, 8), bc_inner=(1, 0, 2), bc_outer=(2, 0, 1))
    if multilevel:
        kw.update(max_level=2, refinement=P.REF_STATIC, regions=[(2, 0.3, 0.5, 0.2, 0.45, 0.3, 0.6)])
    o, g = _pair(oracle_mod, P, **kw)
    rng = np.random.default_rng(11)
    for b in range(o.num_blocks()):
        a = rng.uniform(0.5, 2.0, size=(5, 12, 12, 12))
        o.set_state_full(b, a)
        g.set_state_full(b, a)
    o.exchange()
    g.exchange()
    for b in range(o.num_blocks()):
        assert np.array_equal(g.get_state_full(b), o.get_state_full(b)), b


def test_uniform_state_bitwise(P):
    g = P.Mesh(mesh_nx=(32, 32, 32), block_nx=(16, 16, 16), max_level=1, refinement=P.REF_STATIC,
               regions=[(1, 0.1, 0.4, 0.5, 0.7, 0.2, 0.3)])
    U = np.array([1.3, 1.3 * 0.3, -1.3 * 0.7, 1.3 * 0.11, 2.0])
    for b in range(g.num_blocks()):
        g.set_state(b, np.broadcast_to(U[:, None, None, None], (5, 16, 16, 16)))
    g.refresh()
    g.step(5)
    for b in range(g.num_blocks()):
        S = g.get_state(b)
        for v in range(5):
            assert np.all(S[v] == U[v]), (b, v)


def test_pack_size_invariance(P):
    outs = []
    for ps in (0, 1, 3):
        g = P.Mesh(mesh_nx=(32, 32, 32), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3, pack_size=ps)
        g.set_problem(P.BLAST, [10.0, 0.1, 0.2])
        g.step(4)
        outs.append(gather(g))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_step_host_matches_step(P):
    import torch
    kw = dict(mesh_nx=(32, 32, 32), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3)
    g = P.Mesh(**kw)
    g.set_problem(P.BLAST, [10.0, 0.1, 0.2])
    init = gather(g)
    g.step(3)
    ref = gather(g)
    h = P.Mesh(**kw)
    hin = torch.from_numpy(init.copy()).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    h.step_host(hin, hout, 3)
    torch.cuda.synchronize()
    assert np.array_equal(hout.numpy(), ref)
    # asynchronous problems alternating over two meshes on two streams give the same answers
    a, b = P.Mesh(**kw), P.Mesh(stream=torch.cuda.Stream(), **kw)
    outs = [torch.empty_like(hin).pin_memory() for _ in range(4)]
    for s in range(4):
        M = (a, b)[s % 2]
        if s >= 2:
            M.sync()
        M.step_host_async(hin, outs[s], 3)
    a.sync()
    b.sync()
    for o in outs:
        assert np.array_equal(o.numpy(), ref)


def test_negative_pressure_is_reported(P):
    g = P.Mesh(mesh_nx=(16, 16, 16), block_nx=(16, 16, 16))
    U = np.broadcast_to(np.array([1.0, 0.0, 0.0, 0.0, 1.0])[:, None, None, None], (5, 16, 16, 16)).copy()
    U[4, 3, 4, 5] = -1.0
    g.set_state(0, U)
    with pytest.raises(P.PhError) as e:
        g.refresh()
    assert e.value.code == 6 and "(3,4,5)" in str(e.value)


def test_config2a_full_size_parity(oracle_mod, P):
    """BASELINE config 2 (reading 2a): 256^3 mesh of 64^3 blocks, blast, 10 cycles, all blocks per launch."""
    kw = dict(mesh_nx=(256,) * 3, block_nx=(64,) * 3, xmin=(-.5,) * 3, xmax=(.5,) * 3)
    o, g = _run_both(oracle_mod, P, P.BLAST, [10.0, 0.1, 0.1], 10, **kw)
    _check_run(o, g)


@pytest.mark.parametrize("bc", [0, 1])
def test_direct_halo_equals_materialised_ghosts(P, bc):
    """The direct-halo path (stage kernel reads local neighbour interiors) is bitwise identical to
    the paper's scheme of exchanging every ghost each stage."""
    kw = dict(mesh_nx=(64, 32, 48), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3,
              bc_inner=(bc,) * 3, bc_outer=(bc,) * 3)
    outs = []
    for dh in (True, False):
        g = P.Mesh(direct_halo=dh, **kw)
        assert g.plan_info()["direct_halo"] == dh
        g.set_problem(P.BLAST, [10.0, 0.1, 0.2, 0.05, -0.1, 0.0])
        g.step(6)
        outs.append((gather(g), g.history()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1][:, :2], outs[1][1][:, :2])


def test_graph_replay_equals_eager(P, monkeypatch):
    """one captured cycle replayed N times == N eager cycles (bitwise)"""
    kw = dict(mesh_nx=(32, 32, 32), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3,
              bc_inner=(1, 0, 2), bc_outer=(2, 0, 1))
    outs = []
    for nog in ("0", "1"):
        monkeypatch.setenv("PH_NO_GRAPH", nog)
        g = P.Mesh(**kw)
        g.set_problem(P.BLAST, [10.0, 0.1, 0.2])
        g.step(3)
        g.step(2, 0.0)
        outs.append((gather(g), g.history(), g.launch_count()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]


@pytest.mark.parametrize("recon", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("nseg", [None, "1", "7"])
def test_high_order_blast_and_sod(oracle_mod, P, recon, nseg, monkeypatch):
    """NEXT 3: PPM / WENO-Z (nghost 3) through the generic high-order GPU path vs the oracle.
    This path computes in the oracle's exact operation order (WENO-Z weights and the PPM extremum
    switch amplify round-off), so the states and dt must agree bit for bit.  nseg forces the number
    of segments each line of faces is split into by the line-march flux kernel (None: its own
    choice, which is many short segments at these sizes; "1": one march over the whole line, the
    case of large meshes; "7": segment boundaries at ragged offsets)."""
    if nseg is not None:  # the line march in every direction, with a forced segment count
        monkeypatch.setenv("PH_HO_LINE", "1")
        monkeypatch.setenv("PH_HO_NSEG", nseg)
    o, g = _run_both(oracle_mod, P, P.BLAST, [10.0, 0.1, 0.15], 8, recon=recon, nghost=3,
                     mesh_nx=(48, 48, 48), block_nx=(16, 16, 16), xmin=(-.5,) * 3, xmax=(.5,) * 3)
    _check_run(o, g)
    assert np.array_equal(gather(g), gather(o)) and g.time() == o.time()
    if nseg is not None and recon in (1, 2):
        return  # the 1-D Sod run below adds nothing for these two beyond minmod's
    kw = dict(mesh_nx=(128, 6, 6), block_nx=(32, 6, 6), gamma=1.4, recon=recon, nghost=3,
              bc_inner=(P.OUTFLOW, 0, 2), bc_outer=(P.OUTFLOW, 0, 2))
    o, g = _run_both(oracle_mod, P, P.SOD, [0.5], 100000, tlim=0.1, **kw)
    _check_run(o, g)
    assert np.array_equal(gather(g), gather(o)) and g.time() == o.time()


_STRICT_SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, 'tests')
import paper_2202_12309_b200 as P
import oracle as O
from parity import diagnostics, gather
kw = dict(mesh_nx=(32, 32, 32), block_nx=(32, 32, 32))
g, o = P.Mesh(device=0, **kw), O.Mesh(**kw)
for m in (g, o):
    m.set_problem(P.LINEAR_WAVE, [1e-6, 1, 1, 1])
    m.step(10)
print(json.dumps({"diag": diagnostics(gather(g), gather(o)), "dt": [g.time()[1], o.time()[1]]}))
"""


def test_strict_build_config1_unfloored(oracle_mod, P):
    """SURVEY §8(c) c.3 strict diagnostic build: no FMA contraction, IEEE division / square root and
    the oracle's division by dx (the round-1 stage kernel with the general RK finish).  Config 1's
    fluxes then agree with the oracle's to the last bit or two, so every variable -- the momenta
    included -- meets 1e-12 *without* the momentum floor of reading A27' (un-floored |g-o|/|o|)."""
    import json
    import os
    import subprocess
    import sys
    from paper_2202_12309_b200 import _build
    lib = _build.build_strict()
    env = dict(os.environ, PH_LIB=lib, PH_STAGE_V1="1", PH_NO_HBASE="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", _STRICT_SCRIPT], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    print("strict config 1:", res)
    for v, d in res["diag"].items():
        assert d["rel_unfloored"] <= 1e-12 and d["zero_ref_nonzero_gpu"] == 0, (v, d)
    assert abs(res["dt"][0] - res["dt"][1]) <= 1e-14 * res["dt"][1]
