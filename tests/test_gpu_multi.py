"""Multi-GPU parity through torchrun (NCCL and peer-memory halo); needs >= 2 GPUs (gpurun --gpus 2), else skipped."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [(c, "auto") for c in ("smr2", "smr3_walls", "amr2", "wenoz")] + [("amr16", "peer")]
# multilevel and adaptive meshes with the NCCL halo too (auto picks peer memory for them: an AMR remesh
# rebuilds the peer regions)
CASES += [(c, "nccl") for c in ("smr2", "smr3_walls", "amr2")]
# uniform meshes: both halo transports (NCCL pack/send/unpack, and peer memory read in place)
CASES += [(c, h) for c in ("blast", "sod_walls", "wave64", "tiny") for h in ("nccl", "peer")]
# the fused put: the boundary blocks' stage kernel stores its faces into the peers' buffers itself
CASES += [("blast", "peer-fused"), ("sod_walls", "peer-fused")]


def _run(world, cases, fused):
    """One torchrun process group runs a whole shard of cases (the process start, CUDA context and
    NCCL bootstrap are paid once per shard instead of once per case)."""
    for attempt in range(4):  # the free-port probe can race with another rendezvous: retry
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()),
               os.path.join(ROOT, "tools", "multi_check.py"),
               "--cases", ",".join(f"{c}:{h.split('-')[0]}" for c, h in cases)]
        env = dict(os.environ, PH_FUSED_PUT="1") if fused else None
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT, env=env)
        if "EADDRINUSE" not in r.stderr:
            break
    lines = [l for l in r.stdout.splitlines() if l.startswith("MULTI_CHECK")]
    assert r.returncode == 0 and len(lines) == len(cases), r.stdout[-3000:] + r.stderr[-3000:]
    for l in lines:
        assert '"ok": true' in l, l


# shards: multilevel / AMR / high order, uniform with both transports, the fused put (own env)
SHARDS = {
    "multilevel": [c for c in CASES if c[0] in ("smr2", "smr3_walls", "amr2", "amr16", "wenoz")],
    "uniform": [c for c in CASES if c[0] in ("blast", "sod_walls", "wave64", "tiny") and c[1] != "peer-fused"],
    "fused": [c for c in CASES if c[1] == "peer-fused"],
}


@pytest.mark.parametrize("shard", sorted(SHARDS))
@pytest.mark.parametrize("world", [2, 4])
def test_multi_gpu_matches_oracle_and_single_gpu(shard, world):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    _run(world, SHARDS[shard], shard == "fused")
