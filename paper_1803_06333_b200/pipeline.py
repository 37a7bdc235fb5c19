"""Out-of-core training: chunk keys and the double-buffered streaming pipeline.

Reference: pipeline.py:25-340. `generate_keys` / `keys_to_permutation` are
bit-exact device versions of pipeline.py:29-78 (csrc/prng.cu ChunkKeys).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L

KEY_BLOCK = 4096
STAGE_TIMEOUT_S = 120.0


def _D():
    from . import _device
    return _device


def generate_keys_device(seed, n):
    D = _D()
    out = torch.empty(max(n, 1), dtype=torch.uint32, device=D.device())
    if n > 0:
        L.check(L.lib().glm_chunk_keys(int(seed) & ((1 << 64) - 1), n, D.ptr(out), D.sptr()),
                "glm_chunk_keys")
    return out[:n]


def generate_keys(seed, n, n_threads=1):
    """n 32-bit keys in fixed 4096-wide blocks (pipeline.py:29-73), on the GPU;
    identical for every thread count by construction."""
    if n <= 0:
        return np.empty(0, dtype=np.uint32)
    return _D().to_host(generate_keys_device(seed, n)).astype(np.uint32)


def keys_to_permutation(keys):
    """Stable argsort of the keys (pipeline.py:76-78), on the GPU."""
    from .solver import argsort_u32_device
    k = _D().to_device(np.asarray(keys, dtype=np.uint32), torch.uint32) \
        if not isinstance(keys, torch.Tensor) else keys
    return _D().to_host(argsort_u32_device(k)).astype(np.int64)
