"""Host mirror of the reference's workload generators (proj/include/bht/keygen.hpp, proj/src/keygen.cpp) over the C ABI
(csrc/workload.cu): same names, same arguments, element-for-element the same outputs."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .table import _as_u32, _check, _stream_ptr


@dataclass
class KeySet:
    """key_set (keygen.hpp:13-18): unique sentinel-free keys and the seed that drew them."""
    keys: "torch.Tensor | np.ndarray"
    seed: int = 0

    def size(self) -> int:
        return int(self.keys.numel() if isinstance(self.keys, torch.Tensor) else self.keys.size)


@dataclass
class Queries:
    """vector<query> (keygen.hpp:30-34) as three host arrays."""
    keys: np.ndarray              # uint32
    expected_value: np.ndarray    # uint32; meaningful where expected_present
    expected_present: np.ndarray  # bool


def generate_keys(seed: int, n: int, device: Optional[int] = None, on_device: bool = True, stream=None) -> KeySet:
    """generate_keys (keygen.cpp:50-64): n unique keys by rejection from std::mt19937_64(seed), in stream order."""
    lib = _lib.load()
    device = torch.cuda.current_device() if device is None else device
    if on_device:
        keys = torch.empty(n, dtype=torch.uint32, device=f"cuda:{device}")
        _check(lib.bht_generate_keys(seed, n, keys.data_ptr(), _lib.MEM_DEVICE, device, _stream_ptr(stream, device)))
    else:
        keys = np.empty(n, dtype=np.uint32)
        _check(lib.bht_generate_keys(seed, n, keys.ctypes.data, _lib.MEM_HOST, device, _stream_ptr(stream, device)))
    return KeySet(keys, seed)


def generate_queries(keys, positive_ratio: float, q: int, seed: int, device: Optional[int] = None) -> Queries:
    """generate_queries (keygen.cpp:66-98).  ``keys``: a KeySet or an array / tensor of unique keys.  Raises
    ValueError where the reference throws invalid_argument (ratio outside [0, 1], more positives than keys)."""
    lib = _lib.load()
    arr = keys.keys if isinstance(keys, KeySet) else keys
    kp, kn, kspace, _keep = _as_u32(arr, "keys")
    if device is None:
        device = arr.device.index if isinstance(arr, torch.Tensor) and arr.is_cuda else torch.cuda.current_device()
    out_k = np.empty(q, dtype=np.uint32)
    out_v = np.empty(q, dtype=np.uint32)
    out_p = np.empty(q, dtype=np.uint8)
    _check(lib.bht_generate_queries(kp, kn, kspace, float(positive_ratio), q, seed, out_k.ctypes.data, out_v.ctypes.data,
                                    out_p.ctypes.data, device))
    return Queries(out_k, out_v, out_p.astype(bool))


def save_keys(path: str, keys) -> None:
    """save_keys (keygen.cpp:100-112): flat binary file of little-endian 32-bit keys."""
    arr = keys.keys if isinstance(keys, KeySet) else keys
    if isinstance(arr, torch.Tensor):
        arr = arr.cpu().numpy()
    arr = np.ascontiguousarray(arr).view(np.uint32)
    _check(_lib.load().bht_save_keys(str(path).encode(), arr.ctypes.data, arr.size))


def load_keys(path: str, seed: int = 0) -> KeySet:
    """load_keys (keygen.cpp:114-125)."""
    lib = _lib.load()
    cnt = C.c_uint64()
    _check(lib.bht_load_keys(str(path).encode(), None, 0, C.byref(cnt)))
    out = np.empty(cnt.value, dtype=np.uint32)
    _check(lib.bht_load_keys(str(path).encode(), out.ctypes.data, out.size, C.byref(cnt)))
    return KeySet(out, seed)
