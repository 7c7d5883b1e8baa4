"""Query-shard partitioner: bounds arithmetic and world_size-2 gloo runs
(broadcast of layout buffers, local shards, ordered root gather).  The CPU
test plugs the C oracle in as the compute step; the GPU test (-m gpu) plugs
the CUDA path (DeviceStore + predict_device, FAST tiled) into the same
runner, both ranks on cuda:0, and checks the gathered result bitwise against
one single-process call."""

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


def _worker(rank, world, port, result_q, gpu=False):
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
        n, m = (300_000, 20_001) if gpu else (3000, 1001)
        runner = QueryShardedRunner(dist, torch.device("cpu"), align=256 if gpu else 64)
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
            if gpu:  # the CUDA path: the broadcast bytes -> HBM -> K2 FAST on this rank's shard
                import paper_1402_4986_b200 as il
                from paper_1402_4986_b200.device import DeviceStore, predict_device

                dbufs = [b.to("cuda:0") for b in buffers]
                ds = DeviceStore.from_tensors(LayoutKind(meta.kind), Precision(meta.precision), meta.count,
                                              dbufs, meta.nbytes, 0)
                out = torch.empty(qxl.numel(), dtype=torch.float32, device="cuda:0")
                predict_device(ds, qxl.to("cuda:0"), qyl.to("cuda:0"), out, il.Params(),
                               il.ExecConfig(mode="fast"), "tiled")
                torch.cuda.synchronize()
                return out.cpu()
            raw = buffers[0].numpy()[: meta.nbytes[0]].copy()
            st = LayoutStore(LayoutKind(meta.kind), Precision(meta.precision), meta.count,
                             [raw], __import__("paper_1402_4986_b200.layouts", fromlist=["x"]).buffer_shapes(
                                 LayoutKind(meta.kind), Precision(meta.precision), meta.count))
            q = np.column_stack([qxl.numpy(), qyl.numpy()])
            return torch.from_numpy(oracle.predict(st, q))

        qxf, qyf = (qx.astype(np.float32), qy.astype(np.float32)) if gpu else (qx, qy)
        full = runner.run(compute, bufs, meta, torch.from_numpy(qxf[lo:hi]), torch.from_numpy(qyf[lo:hi]), m)
        if rank == 0:
            x, y, z = generate_cloud_arrays(n, 0)
            st = LayoutStore.from_arrays(x, y, z, LayoutKind.AoaS, Precision.single)
            if gpu:
                import paper_1402_4986_b200 as il

                ref = il.run_tiled(st, np.column_stack([qx, qy]), il.Params(), il.ExecConfig(mode="fast"))
                truth = oracle.truth(st, np.column_stack([qx, qy]))
                ok = np.array_equal(full.numpy(), ref) and np.max(np.abs(ref - truth) / truth) <= 1e-5
            else:
                ref = oracle.predict(st, np.column_stack([qx, qy]))
                ok = np.array_equal(full.numpy(), ref)
            result_q.put(bool(ok))
        else:
            assert full is None  # root gather
    finally:
        dist.destroy_process_group()


def _run_world2(gpu):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, gpu)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert q.get() is True


def test_gloo_world2_bit_identical_to_single_process():
    _run_world2(gpu=False)


@pytest.mark.gpu
def test_gloo_world2_cuda_path_bit_identical():
    """Two ranks, each running the CUDA kernels on its 256-aligned query
    shard, gathered to the root == one single-process FAST call, bitwise."""
    _run_world2(gpu=True)
