"""Multi-GPU query partitioner: one process per GPU over torch.distributed.

The reference has no multi-device path; its only parallelism is
static query blocks on a thread pool whose boundaries depend on the workload
alone (strategies.py:15-21,137-145).  ``out[q]`` depends only on query q and
all data (kernels.py:42-67), so the B200 design shards QUERIES:

  1. the data store is replicated by ONE broadcast of its raw layout buffers
     from the source rank (NCCL over NVLink/NVSwitch; gloo in CPU tests),
  2. each rank evaluates its contiguous query shard [lo, hi) on its own GPU,
  3. the per-rank predictions are gathered to the root in rank order (a
     root gather: every rank sends only its own shard).

This is the torchrun (one process per GPU) form of the job.  The drop-in
call itself drives several GPUs from ONE process: ExecConfig(devices=...)
-> idw_params.devices (include/idw_b200.h), with the store broadcast by a
cudaMemcpyPeerAsync tree and each shard copied straight into the caller's
output slice -- same shards (shard_bounds, align 256), same bits.

There is no reduction, so every query keeps its single-device summation
order and results are bit-identical for any world size, in both modes: EXACT
sums in the reference's strict order, and FAST's summation chunks depend on n
alone while its query groups (32*Q consecutive queries) stay whole inside
``align``-query shards (align = 256, a multiple of every group size;
tests/test_determinism_gpu.py checks 1 vs 2/4/8 shards bitwise at C3).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable


def shard_bounds(m: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """Contiguous, near-equal shard of m queries for `rank` of `world`.

    Shard sizes differ by at most `align` queries; boundaries are multiples of
    `align` (except the global end)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if align < 1:
        raise ValueError("align must be >= 1")
    units = -(-m // align)
    base, extra = divmod(units, world)
    lo_u = rank * base + min(rank, extra)
    hi_u = lo_u + base + (1 if rank < extra else 0)
    return min(m, lo_u * align), min(m, hi_u * align)


def padded_shard(m: int, world: int, align: int = 1) -> int:
    """Largest shard length (all_gather needs equal-size chunks)."""
    return max(shard_bounds(m, world, r, align)[1] - shard_bounds(m, world, r, align)[0] for r in range(world))


@dataclass
class StoreMeta:
    kind: str
    precision: str
    count: int
    nbytes: list


class QueryShardedRunner:
    """Broadcast a store, evaluate local query shards, gather predictions.

    ``compute(buffers, meta, qx, qy) -> out`` evaluates the local shard; on GPU
    ranks it wraps libidw_b200 (DeviceStore + predict_device), in CPU tests
    any callable.  Tensors live on ``device`` (cuda:LOCAL_RANK or cpu).
    """

    def __init__(self, dist, device, align: int = 256, src: int = 0):
        self.dist = dist
        self.device = device
        self.align = align
        self.src = src
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()

    # -- 1. replicate the data store ------------------------------------
    def broadcast_meta(self, meta: StoreMeta | None) -> StoreMeta:
        box = [meta]
        self.dist.broadcast_object_list(box, src=self.src)
        return box[0]

    def broadcast_buffers(self, buffers, meta: StoreMeta, pad: int = 64):
        """Replicate raw layout buffers (uint8) from src; returns local tensors.
        Each buffer carries `pad` spare bytes (bulk-copy tail rounding)."""
        import torch

        out = []
        for k, nb in enumerate(meta.nbytes):
            if self.rank == self.src:
                t = buffers[k]
                assert t.dtype == torch.uint8 and t.numel() >= nb
            else:
                t = torch.zeros(nb + pad, dtype=torch.uint8, device=self.device)
            self.dist.broadcast(t, src=self.src)
            out.append(t)
        return out

    # -- 2. local shard ---------------------------------------------------
    def bounds(self, m: int) -> tuple[int, int]:
        return shard_bounds(m, self.world, self.rank, self.align)

    # -- 3. gather --------------------------------------------------------
    def gather(self, local, m: int):
        """Root gather of the shards in rank order (each rank sends only its
        own predictions: m values reach the root once, not world x m as an
        all-gather would).  Returns the full vector on the root, None
        elsewhere.  Shards are padded to equal length for the collective."""
        import torch

        L = padded_shard(m, self.world, self.align)
        # gloo gathers host tensors; NCCL gathers in place on the GPUs
        on = local.device if self._backend() == "nccl" else torch.device("cpu")
        buf = torch.zeros(L, dtype=local.dtype, device=on)
        buf[: local.numel()].copy_(local)
        parts = [torch.empty_like(buf) for _ in range(self.world)] if self.rank == self.src else None
        self.dist.gather(buf, gather_list=parts, dst=self.src)
        if self.rank != self.src:
            return None
        out = []
        for r in range(self.world):
            lo, hi = shard_bounds(m, self.world, r, self.align)
            out.append(parts[r][: hi - lo])
        return torch.cat(out)

    def _backend(self) -> str:
        try:
            return str(self.dist.get_backend())
        except Exception:  # pragma: no cover
            return "gloo"

    # -- whole job ----------------------------------------------------------
    def run(self, compute: Callable, buffers, meta: StoreMeta, qx_local, qy_local, m: int):
        out_local = compute(buffers, meta, qx_local, qy_local)
        return self.gather(out_local, m)
