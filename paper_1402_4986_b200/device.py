"""HBM-resident stores and the asynchronous device entry point.

``DeviceStore`` uploads a LayoutStore's raw buffers once (byte-identical, each
padded by 64 bytes so the tail tile's 16-byte-rounded bulk copy stays inside
the allocation) and keeps them resident; ``predict_device`` launches one
strategy over device query/output tensors on the current torch stream without
synchronising.  torch is plumbing here (allocation, streams); the compute is
libidw_b200.
"""

from __future__ import annotations

import numpy as np

from . import _capi
from .core import Params
from .strategies import ExecConfig

PAD = 64


class DeviceStore:
    def __init__(self, store, device: int = 0):
        import torch

        self.kind = store.kind
        self.precision = store.precision
        self.count = store.count
        self.shapes = getattr(store, "shapes", None)
        self.stats = store.stats
        self.device = device
        dev = torch.device("cuda", device)
        self.tensors = []
        for buf in store.buffers:
            host = np.ascontiguousarray(buf).view(np.uint8)
            t = torch.zeros(host.nbytes + PAD, dtype=torch.uint8, device=dev)
            t[: host.nbytes].copy_(torch.from_numpy(host))
            self.tensors.append(t)
        self.nbytes = [np.ascontiguousarray(b).nbytes for b in store.buffers]

    @classmethod
    def from_tensors(cls, kind, precision, count, tensors, nbytes, device: int = 0, stats=None):
        """Wrap already-resident uint8 buffers (e.g. received by broadcast)."""
        self = cls.__new__(cls)
        self.kind, self.precision, self.count = kind, precision, count
        self.shapes = None
        self.stats = stats
        self.device = device
        self.tensors = list(tensors)
        self.nbytes = list(nbytes)
        return self

    # -- device-side packers / converters / dump loader (§8f rows) -----------
    @classmethod
    def _alloc(cls, kind, precision, count, device, stats=None):
        import torch

        from .layouts import AccessStats, buffer_shapes

        shapes = buffer_shapes(kind, precision, count)
        dev = torch.device("cuda", device)
        tensors = [torch.zeros(sh.nbytes + PAD, dtype=torch.uint8, device=dev) for sh in shapes]
        self = cls.from_tensors(kind, precision, count, tensors, [sh.nbytes for sh in shapes], device,
                                stats or AccessStats(precision.itemsize))
        self.shapes = shapes
        return self

    @classmethod
    def from_arrays(cls, x, y, z, kind, precision, device: int = 0):
        """Pack fp64 component arrays on the GPU (idw_pack_device): the same
        bytes as LayoutStore.from_arrays (reference layouts.py:172-186)."""
        import torch

        from .layouts import check_legal

        check_legal(kind, precision)
        dev = torch.device("cuda", device)
        comps = [torch.as_tensor(np.asarray(a, dtype=np.float64)).to(dev) for a in (x, y, z)]
        n = int(comps[0].numel())
        if n == 0:
            raise ValueError("no data points")
        self = cls._alloc(kind, precision, n, device)
        _capi.pack_device(comps[0].data_ptr(), comps[1].data_ptr(), comps[2].data_ptr(), n, self.native(), device,
                          torch.cuda.current_stream(dev).cuda_stream)
        return self

    def convert(self, target):
        """Re-layout on the GPU (idw_convert_device), value-preserving like
        LayoutStore.convert (reference layouts.py:251-255)."""
        import torch

        from .layouts import check_legal

        check_legal(target, self.precision)
        out = DeviceStore._alloc(target, self.precision, self.count, self.device)
        _capi.convert_device(self.native(), out.native(), self.device,
                             torch.cuda.current_stream(self.device).cuda_stream)
        return out

    def to_host(self):
        """Copy the raw buffers back into a host LayoutStore (byte-exact)."""
        from .layouts import LayoutStore, aligned_zeros, buffer_shapes

        shapes = buffer_shapes(self.kind, self.precision, self.count)
        bufs = []
        for t, sh in zip(self.tensors, shapes):
            b = aligned_zeros(sh.nbytes)
            b[:] = t[: sh.nbytes].cpu().numpy()
            bufs.append(b)
        return LayoutStore(self.kind, self.precision, self.count, bufs, shapes)

    @classmethod
    def from_dump(cls, path, device: int = 0):
        """Load an IDWL dump (reference layouts.py:257-294: <4sBBQ> header +
        raw buffers) straight into device buffers, skipping the host repack."""
        import torch

        from .layouts import DUMP_HEADER, DUMP_MAGIC, KIND_CODE, PRECISION_CODE, buffer_shapes

        with open(path, "rb") as fh:
            blob = fh.read()
        if len(blob) < DUMP_HEADER.size:
            raise ValueError("truncated layout dump")
        magic, kcode, pcode, count = DUMP_HEADER.unpack_from(blob)
        if magic != DUMP_MAGIC:
            raise ValueError("bad magic; not a layout dump")
        kinds = {v: k for k, v in KIND_CODE.items()}
        precs = {v: k for k, v in PRECISION_CODE.items()}
        if kcode not in kinds or pcode not in precs:
            raise ValueError("unknown layout or precision code")
        kind, precision = kinds[kcode], precs[pcode]
        shapes = buffer_shapes(kind, precision, count)
        if len(blob) != DUMP_HEADER.size + sum(sh.nbytes for sh in shapes):
            raise ValueError("layout dump has wrong size")
        self = cls._alloc(kind, precision, count, device)
        pos = DUMP_HEADER.size
        for t, sh in zip(self.tensors, shapes):
            host = torch.frombuffer(bytearray(blob[pos:pos + sh.nbytes]), dtype=torch.uint8)
            t[: sh.nbytes].copy_(host)
            pos += sh.nbytes
        return self

    @property
    def dtype(self):
        import torch

        return torch.float64 if self.precision.value == "double" else torch.float32

    def native(self) -> _capi.IdwStore:
        return _capi.make_store(self.kind.value, self.precision.value, self.count,
                                [t.data_ptr() for t in self.tensors], self.nbytes)


def predict_device(dstore: DeviceStore, qx, qy, out, params: Params = Params(),
                   cfg: ExecConfig | None = None, variant: str = "tiled", stream=None):
    """Launch ``variant`` for device tensors qx, qy -> out (run dtype, contiguous)
    on ``stream`` (default: torch's current stream).  Returns the native stats.
    ``cfg.devices`` (starting with the store's device) spreads the call over
    several GPUs: peer-copy broadcast of the store, query shards out and
    predictions back by peer copies; ``stream`` waits for all of them."""
    import torch

    cfg = cfg or ExecConfig()
    m = int(out.shape[0])
    if stream is None:
        stream = torch.cuda.current_stream(dstore.device)
    if cfg.devices and cfg.devices[0] != dstore.device:
        raise ValueError(f"device list must start with the store's device {dstore.device}")
    prm = _capi.make_params(params.p, params.zero_eps, variant, cfg.mode, cfg.group_size,
                            cfg.tile_size, cfg.splits, dstore.device, cfg.devices)
    return _capi.run_device(dstore.native(), qx.data_ptr(), qy.data_ptr(), m, prm,
                            out.data_ptr(), stream.cuda_stream)


class DevicePlan:
    """``predict_device`` captured once into a CUDA graph (idw_plan_create) and
    replayed per batch: the serving loop refills ``qx``/``qy`` in place and
    calls :meth:`launch` -- one graph launch instead of a runtime call per
    kernel.  Holds references to the tensors whose pointers the graph uses."""

    def __init__(self, dstore: DeviceStore, qx, qy, out, params: Params = Params(),
                 cfg: ExecConfig | None = None, variant: str = "tiled"):
        cfg = cfg or ExecConfig()
        self._keep = (dstore, qx, qy, out)
        prm = _capi.make_params(params.p, params.zero_eps, variant, cfg.mode, cfg.group_size,
                                cfg.tile_size, cfg.splits, dstore.device)
        self._plan = _capi.Plan(dstore.native(), qx.data_ptr(), qy.data_ptr(), int(out.shape[0]), prm,
                                out.data_ptr())
        self.launches = self._plan.launches
        self.device = dstore.device

    def launch(self, stream=None) -> None:
        import torch

        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self._plan.launch(stream.cuda_stream)

    def kernel_ms(self) -> tuple[float, float]:
        """(variant kernels ms, fix-up ms) of the most recent launch."""
        return self._plan.kernel_ms()

    def close(self) -> None:
        self._plan.close()
