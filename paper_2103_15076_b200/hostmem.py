"""Pinned host buffers for the numpy API.

Results handed back as numpy arrays are allocated in page-locked memory
(torch's caching host allocator, wrapped zero-copy as numpy): the library's
fused result-emission kernel writes them directly through their mapped device
addresses, and the remaining copies run at full PCIe/C2C rate instead of being
staged through a pageable bounce buffer; arrays passed back in (e.g. features
pooled level by level) are then pinned too.  The allocator caches freed blocks, so repeated
calls do not pay cudaHostAlloc.  Without a usable CUDA runtime this falls back
to ordinary numpy allocations (the compute path itself still requires the GPU).
"""

import numpy as np

_TORCH_DT = None
_ok = None


def _torch():
    global _ok, _TORCH_DT
    if _ok is None:
        try:
            import torch

            _ok = bool(torch.cuda.is_available())
            _TORCH_DT = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
                         np.dtype(np.int64): torch.int64, np.dtype(np.int32): torch.int32}
        except Exception:  # pragma: no cover
            _ok = False
    return _ok


def empty(shape, dtype) -> np.ndarray:
    dtype = np.dtype(dtype)
    if _torch() and dtype in _TORCH_DT:
        import torch

        return torch.empty(tuple(shape), dtype=_TORCH_DT[dtype], pin_memory=True).numpy()
    return np.empty(shape, dtype=dtype)
