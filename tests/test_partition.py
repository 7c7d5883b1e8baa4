"""Query-shard partitioner: bounds arithmetic and a world_size-2 gloo run on
CPU (broadcast of layout buffers, local shards, ordered gather).  The compute
callback is the C oracle here -- the GPU path plugs libidw_b200 into the same
runner (bench.py)."""

import os
import socket

import numpy as np
import pytest

from paper_1402_4986_b200.partition import padded_shard, shard_bounds


@pytest.mark.parametrize("m", [0, 1, 7, 255, 256, 1000, 1 << 20])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("align", [1, 32, 256])
def test_shards_cover_exactly_once(m, world, align):
    cover = []
    sizes = []
    for r in range(world):
        lo, hi = shard_bounds(m, world, r, align)
        assert 0 <= lo <= hi <= m
        if r:
            assert lo == prev_hi  # noqa: F821 - contiguous, rank order
        prev_hi = hi  # noqa: F841
        cover.append((lo, hi))
        sizes.append(hi - lo)
        if hi < m:
            assert hi % align == 0
    assert cover[0][0] == 0 and cover[-1][1] == m
    assert max(sizes) - min(sizes) <= (align if m % align == 0 else 2 * align)
    assert padded_shard(m, world, align) == max(sizes)


def test_bad_args():
    with pytest.raises(ValueError):
        shard_bounds(10, 0, 0)
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 0, align=0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    import torch
    import torch.distributed as dist

    import oracle
    from paper_1402_4986_b200.generator import generate_cloud_arrays
    from paper_1402_4986_b200.layouts import LayoutKind, LayoutStore
    from paper_1402_4986_b200.core import Precision
    from paper_1402_4986_b200.partition import QueryShardedRunner, StoreMeta

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, m = 3000, 1001
        runner = QueryShardedRunner(dist, torch.device("cpu"), align=64)
        bufs, meta = None, None
        if rank == 0:  # only the source rank holds the data
            x, y, z = generate_cloud_arrays(n, 0)
            st = LayoutStore.from_arrays(x, y, z, LayoutKind.AoaS, Precision.single)
            meta = StoreMeta(st.kind.value, st.precision.value, st.count, [b.nbytes for b in st.buffers])
            bufs = [torch.from_numpy(np.concatenate([b, np.zeros(64, np.uint8)])) for b in st.buffers]
        meta = runner.broadcast_meta(meta)
        bufs = runner.broadcast_buffers(bufs, meta)
        qx, qy, _ = generate_cloud_arrays(m, 1)
        lo, hi = runner.bounds(m)

        def compute(buffers, meta, qxl, qyl):
            raw = buffers[0].numpy()[: meta.nbytes[0]].copy()
            st = LayoutStore(LayoutKind(meta.kind), Precision(meta.precision), meta.count,
                             [raw], __import__("paper_1402_4986_b200.layouts", fromlist=["x"]).buffer_shapes(
                                 LayoutKind(meta.kind), Precision(meta.precision), meta.count))
            q = np.column_stack([qxl.numpy(), qyl.numpy()])
            return torch.from_numpy(oracle.predict(st, q))

        full = runner.run(compute, bufs, meta, torch.from_numpy(qx[lo:hi]), torch.from_numpy(qy[lo:hi]), m)
        if rank == 0:
            x, y, z = generate_cloud_arrays(n, 0)
            st = LayoutStore.from_arrays(x, y, z, LayoutKind.AoaS, Precision.single)
            ref = oracle.predict(st, np.column_stack([qx, qy]))
            result_q.put(bool(np.array_equal(full.numpy(), ref)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_bit_identical_to_single_process():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert q.get() is True
