"""Device plumbing: the CUDA device, stream and tensor conversions.

PyTorch is used only for device memory, streams and host<->device copies;
every compute step goes through libbytestore_b200.so.  There is no CPU
fallback: without a CUDA device the device path raises.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

__all__ = ["device", "require_cuda", "to_dev_i64", "to_dev_u64", "to_dev_u8", "to_dev_u32",
           "host_u32", "host_u64", "stream"]


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2209_00220_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    _lib.load()


def device() -> torch.device:
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    return _lib.stream_ptr()


def _to_dev(x, np_dtype, view_dtype, torch_dtype):
    dev = device()
    if isinstance(x, torch.Tensor):
        t = x
        if t.dtype != torch_dtype:
            if torch_dtype == torch.int64 and t.dtype in (torch.int32, torch.int16, torch.uint8,
                                                          torch.int8):
                t = t.to(torch.int64)
            elif t.element_size() == torch.empty(0, dtype=torch_dtype).element_size():
                t = t.view(torch_dtype)
            else:
                t = t.to(torch_dtype)
        return t.to(dev, non_blocking=True).contiguous()
    a = np.ascontiguousarray(np.asarray(x).astype(np_dtype, copy=False))
    return torch.from_numpy(a.view(view_dtype)).to(dev, non_blocking=False)


def to_dev_i64(x) -> torch.Tensor:
    return _to_dev(x, np.int64, np.int64, torch.int64)


def to_dev_u64(x) -> torch.Tensor:
    """uint64 codes stored bit-for-bit in an int64 tensor."""
    if isinstance(x, torch.Tensor):
        return _to_dev(x, np.uint64, np.int64, torch.int64)
    a = np.asarray(x)
    if a.dtype.kind == "i" and (a < 0).any():
        raise ValueError("codes must be non-negative")
    return _to_dev(a.astype(np.uint64), np.uint64, np.int64, torch.int64)


def to_dev_u8(x) -> torch.Tensor:
    return _to_dev(x, np.uint8, np.uint8, torch.uint8)


def to_dev_u32(x) -> torch.Tensor:
    """uint32 words stored bit-for-bit in an int32 tensor."""
    return _to_dev(x, np.uint32, np.int32, torch.int32)


def host_u32(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


def host_u64(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)
