"""Device plumbing: torch tensors as raw device pointers and stream handles.

PyTorch only provides memory, streams and copies here; every computation on
the re-sampling path is a kernel of ``liblcb200.so``.
"""

from __future__ import annotations

import numpy as np
import torch


def device(dev=None) -> torch.device:
    if dev is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2604_17353_b200 needs a CUDA device (no CPU fallback)")
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(dev)
    if d.type != "cuda":
        raise RuntimeError("paper_2604_17353_b200 runs on CUDA devices only")
    return d


def stream_ptr(dev=None) -> int:
    return torch.cuda.current_stream(device(dev)).cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def to_dev(x, dtype, dev) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.asarray(x), dtype=dtype).to(dev).contiguous()


def u64_tensor(values, dev) -> torch.Tensor:
    """uint64 digests/seeds carried in an int64 tensor (bit pattern preserved)."""
    a = np.asarray(values, dtype=np.uint64).view(np.int64)
    return torch.from_numpy(a.copy()).to(dev)


def u64_numpy(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)
