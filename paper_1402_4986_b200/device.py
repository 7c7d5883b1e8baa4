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
    on ``stream`` (default: torch's current stream).  Returns the native stats."""
    import torch

    cfg = cfg or ExecConfig()
    m = int(out.shape[0])
    if stream is None:
        stream = torch.cuda.current_stream(dstore.device)
    prm = _capi.make_params(params.p, params.zero_eps, variant, cfg.mode, cfg.group_size,
                            cfg.tile_size, cfg.splits, dstore.device)
    return _capi.run_device(dstore.native(), qx.data_ptr(), qy.data_ptr(), m, prm,
                            out.data_ptr(), stream.cuda_stream)
