"""Multi-process paths.

* CPU (gloo, world_size 2): the host-side rank plumbing -- IPC-handle
  exchange through torch.distributed and the rank/world bookkeeping used by
  bench.py -- runs without a GPU.
* GPU (>= 2 devices): tests/mgpu_worker.py under torchrun, one rank per GPU,
  checks the NVLink-fused push/pull against the oracle bit-exactly.
"""
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def _gloo_exchange(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    handle = bytes([rank]) * 64  # stands in for a cudaIpcMemHandle_t
    handles = [None] * world
    dist.all_gather_object(handles, handle)
    blob = b"".join(handles)
    q.put((rank, len(blob), blob[::64]))
    dist.destroy_process_group()


def test_ipc_handle_exchange_gloo_world2():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_gloo_exchange, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank sees the handles rank-major, n * ZEN_IPC_HANDLE_BYTES bytes
    assert out == [(0, 128, bytes([0, 1])), (1, 128, bytes([0, 1]))]


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(20000, 64, 0.01), (100000, 64, 0.01)])
def test_bp_multi_gpu_parity(shape):
    n = min(_ngpus(), 4)
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    rows, width, density = shape
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1",
           f"--nproc-per-node={n}", os.path.join(ROOT, "tests", "mgpu_worker.py"),
           str(rows), str(width), str(density)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MGPU OK" in r.stdout


@pytest.mark.gpu
def test_bp_rank_mode_eight_ranks():
    """n = 8 rank mode (the headline node count), one process per GPU, every
    rank mapping the others' arenas over CUDA IPC.  Ranks that spin on each
    other's flags must not share a GPU (time-sliced spinning processes can
    trip a context-switch timeout), so this needs 8 devices; with fewer, the
    n = 8 data path is covered by local mode (tests/test_gpu_fullsize.py)."""
    if _ngpus() < 8:
        pytest.skip("needs 8 GPUs (one rank per GPU)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nnodes=1",
           "--nproc-per-node=8", os.path.join(ROOT, "tests", "mgpu_worker.py"),
           "20000", "64", "0.01"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MGPU OK n=8" in r.stdout
