"""Owner of one libhpgmxp context (one per process / GPU / hierarchy)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .comm import runtime

INFO_KEYS = ("n", "n_ext", "nnz", "ncolors") + tuple(f"off{i}" for i in range(9)) + \
    ("halo", "ld", "nneighbours", "device_bytes")


class Context:
    def __init__(self, domain, levels, nu1=1, nu2=1, nu_c=1, world=None):
        rt = runtime()
        self.device = rt.device
        self.stream = rt.stream
        self.nranks = 1 if world is None else world.nranks
        self.rank = domain.rank
        self.levels = levels
        uid = None
        if self.nranks > 1:
            uid = C.create_string_buffer(world.nccl_uid(), 128)
        h = C.c_void_p()
        L = _lib.lib()
        _lib.check(L.hpg_create(C.byref(h), rt.device.index, domain.rank, self.nranks,
                                _lib.ints(*domain.proc_dims), _lib.ints(*domain.local_dims),
                                levels, nu1, nu2, nu_c, uid, C.c_void_p(rt.stream_ptr)))
        self.h = h
        self._info = [self._level_info(l) for l in range(levels)]

    def call(self, name, *args):
        if self.h is None:
            raise RuntimeError("context already destroyed")
        _lib.check(getattr(_lib.lib(), name)(self.h, *args))

    def _level_info(self, l):
        buf = np.zeros(17, dtype=np.int64)
        self.call("hpg_level_info", l, buf.ctypes.data_as(C.POINTER(C.c_int64)), 17)
        return dict(zip(INFO_KEYS, (int(v) for v in buf)))

    def level_info(self, l):
        return self._info[l]

    def launches(self):
        return int(_lib.lib().hpg_launch_count(self.h))

    def timers(self, mode, seconds=None):
        out = np.zeros(8) if seconds is None else seconds
        self.call("hpg_timers", mode, out.ctypes.data_as(C.POINTER(C.c_double)))
        return out

    def set_option(self, key, value):
        self.call("hpg_set_option", key.encode(), int(value))

    def sync(self):
        self.call("hpg_sync")

    def close(self):
        if self.h is not None:
            _lib.lib().hpg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
