"""Loader for the sm_100a library (libstabgpu.so) and device contexts.

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every entry point raises.  The library is built in-tree by
``__graft_entry__.build()`` (or ``make``) so the python process that imports
this module loads ``paper_1701_03572_b200/libstabgpu.so`` from the repo.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import _abi

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STABGPU_LIB", os.path.join(_HERE, "libstabgpu.so"))

_lib = None
_lock = threading.Lock()
_contexts: dict[int, "Context"] = {}


class StabError(RuntimeError):
    """Base of the error hierarchy (stab::Error, errors.hpp:9-12)."""


class InvalidInputError(StabError):
    pass


class InvalidConfigError(StabError):
    pass


class InvalidTransformError(StabError):
    pass


class DegenerateInputError(StabError):
    pass


class SequencingError(StabError):
    pass


class IoError(StabError):
    pass


class CudaError(StabError):
    pass


_ERRORS = {
    _abi.INVALID_INPUT: InvalidInputError,
    _abi.INVALID_CONFIG: InvalidConfigError,
    _abi.INVALID_TRANSFORM: InvalidTransformError,
    _abi.DEGENERATE_INPUT: DegenerateInputError,
    _abi.SEQUENCING: SequencingError,
    _abi.IO: IoError,
    _abi.CUDA: CudaError,
}


def load() -> C.CDLL:
    """Loads libstabgpu.so (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build the CUDA library first "
                    "(python -c 'import __graft_entry__ as g; g.build()' or `make`); "
                    "there is no CPU fallback")
            _lib = _abi.bind(C.CDLL(LIB_PATH), _abi.PROTOTYPES)
        return _lib


def check(rc: int) -> None:
    if rc != _abi.OK:
        msg = load().stabgpu_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, StabError)(msg)


class Context:
    """One stabgpu_ctx (device, stream, scratch pools)."""

    def __init__(self, device: int = 0):
        lib = load()
        h = C.c_void_p()
        check(lib.stabgpu_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    def close(self) -> None:
        if self.handle:
            load().stabgpu_destroy(self.handle)
            self.handle = C.c_void_p()

    def set_stream(self, stream_ptr: int | None) -> None:
        check(load().stabgpu_set_stream(self.handle, C.c_void_p(stream_ptr or 0)))

    def stats(self) -> _abi.Stats:
        s = _abi.Stats()
        check(load().stabgpu_get_stats(self.handle, C.byref(s)))
        return s

    def read_scratch(self, name: str, dtype, count: int | None = None):
        """Diagnostic: a copy of the named device scratch buffer as numpy."""
        import numpy as np

        have = C.c_size_t(0)
        check(load().stabgpu_debug_read_scratch(self.handle, name.encode(), None, 0, C.byref(have)))
        dt = np.dtype(dtype)
        n = have.value // dt.itemsize if count is None else count
        out = np.zeros(n, dt)
        check(load().stabgpu_debug_read_scratch(self.handle, name.encode(), C.c_void_p(out.ctypes.data),
                                                out.nbytes, None))
        return out

    def enable_timing(self, on: bool = True) -> None:
        check(load().stabgpu_enable_timing(self.handle, 1 if on else 0))


def context(device: int = 0) -> Context:
    with _lock:
        ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _contexts[device] = ctx
    return ctx


def reset_contexts() -> None:
    """Destroys the cached contexts (the next call gets a fresh one with empty
    scratch pools)."""
    with _lock:
        ctxs = list(_contexts.values())
        _contexts.clear()
    for c in ctxs:
        c.close()
