"""world_size-2 torch.distributed (gloo, CPU) test of the multi-GPU sharding path.

Each rank takes its contiguous shard of one global batch (paper_1304_7054_b200
.shard), computes it with the CPU checker (no GPU here), and the shards are
all-gathered: the concatenation must equal the single-process result bit for
bit, and the slices must tile [0, B) exactly -- the same properties the
bench's one-process-per-GPU layout and the runtime's in-process device
sharding rely on. No data-path collective is needed by the product; gloo is
only used here to move the test's results.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1304_7054_b200 import BatchView, MatrixView
from paper_1304_7054_b200.shard import shard_batch, shard_range, sub_batch


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, batch, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.oracle import Oracle

    o = Oracle()
    n = 7
    a, b, _, x, y = o.generate_batch(np.float32, 3, n, False, batch)
    xb = BatchView(MatrixView(x, n, n, n), batch, n * n)
    p0, p1 = shard_range(rank, world, batch)
    mine = shard_batch(xb, rank, world)
    assert mine.batch_count == p1 - p0 and mine.base.offset == p0 * n * n
    cnt = p1 - p0
    xs = x[p0 * n * n:p1 * n * n]
    ys = np.zeros(cnt * n * n, np.float32)
    o.kron2("N", "N", "N", n, n, n, n, cnt, np.float32(1), a, n, b, n, xs, n, n * n, np.float32(0), ys, n, n * n)
    # gather variable-size shards (pad to the max shard)
    per = -(-batch // world)
    buf = torch.zeros(per * n * n)
    buf[:ys.size] = torch.from_numpy(ys)
    parts = [torch.zeros(per * n * n) for _ in range(world)]
    dist.all_gather(parts, buf)
    counts = [torch.zeros(1) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([float(cnt)]))
    if rank == 0:
        full = np.concatenate([p[:int(c.item()) * n * n].numpy() for p, c in zip(parts, counts)])
        ref = np.zeros(batch * n * n, np.float32)
        o.kron2("N", "N", "N", n, n, n, n, batch, np.float32(1), a, n, b, n, x, n, n * n, np.float32(0), ref, n, n * n)
        out_q.put(bool(np.array_equal(full.view(np.uint32), ref.view(np.uint32))))
    dist.barrier()
    dist.destroy_process_group()


def _gpu_worker(rank, world, port, batch, out_q):
    """One process per 'GPU' (both on cuda:0 here): the rank's contiguous shard
    runs through the PRODUCT (kb.kron3, device-resident, the bench's layout),
    the host barrier / result exchange is gloo -- no NCCL, no data-path
    collective."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1304_7054_b200 as kb
    from oracle.oracle import Oracle

    torch.cuda.set_device(0)
    o = Oracle()
    n = 16
    e = n ** 3
    a, b, c, x, y = o.generate_batch(np.float64, 4, n, True, batch)
    p0, p1 = shard_range(rank, world, batch)
    cnt = p1 - p0
    X = torch.from_numpy(x[p0 * e:p1 * e].copy()).cuda()
    Y = torch.zeros(cnt * e, dtype=torch.float64, device="cuda")
    pr = kb.KronProblem3D(m_a=n, n_a=n, m_b=n, n_b=n, m_c=n, n_c=n)
    if cnt:
        kb.kron3(pr, MatrixView(a, n, n, n), MatrixView(b, n, n, n), MatrixView(c, n, n, n),
                 BatchView(kb.Array3View(X, n, n, n, n, n * n), cnt, e),
                 BatchView(kb.Array3View(Y, n, n, n, n, n * n), cnt, e), kb.Workspace(None, cnt * e))
    dist.barrier()  # host barrier between the shards
    per = -(-batch // world)
    buf = torch.zeros(per * e, dtype=torch.float64)
    buf[:cnt * e] = Y.cpu()
    parts = [torch.zeros(per * e, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, buf)
    if rank == 0:
        full = np.concatenate([parts[r][:(shard_range(r, world, batch)[1] - shard_range(r, world, batch)[0]) * e]
                               .numpy() for r in range(world)])
        ref = np.zeros(batch * e)
        o.kron3("N", "N", "N", n, n, n, n, n, n, batch, 1.0, a, n, b, n, c, n, x, n, n * n, e, 0.0, ref, n, n * n, e)
        out_q.put(bool(np.array_equal(full.view(np.uint64), ref.view(np.uint64))))
    dist.barrier()
    dist.destroy_process_group()


def _run_world(target, batch, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert q.get(timeout=5) is True


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [777, 1])
def test_gloo_world2_library_shards_gpu(batch):
    _run_world(_gpu_worker, batch)


@pytest.mark.parametrize("batch", [1001, 2])
def test_gloo_world2_shards_are_bit_identical(batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=5) is True


def test_shard_ranges_tile_the_batch():
    for batch in (0, 1, 7, 1000, 4194304):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(r, world, batch) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and a0 <= a1
    xb = BatchView(MatrixView(np.zeros(100), 3, 3, 3), 10, 10)
    s = sub_batch(xb, 2, 5)
    assert s.batch_count == 3 and s.base.offset == 20 and s.base.len == 80
    with pytest.raises(ValueError):
        shard_range(2, 2, 10)
