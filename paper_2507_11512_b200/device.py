"""Owner of one libhpgmxp context (one per process / GPU / hierarchy)."""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .comm import runtime

INFO_KEYS = ("n", "n_ext", "nnz", "ncolors") + tuple(f"off{i}" for i in range(9)) + \
    ("halo", "ld", "nneighbours", "device_bytes", "zero_sweep_slots", "stencil_rows", "stencil_lower")


BOOL_DEFAULTS = {"stencil": 1, "lower": 0, "graphs": 1, "pdl": 1, "gs_rev": 1}

_LIVE = []  # weak references to the live contexts, newest last (see context_for)


def context_for(device, n, nranks=1):
    """A live context on ``device`` whose level 0 has ``n`` rows (the newest such),
    else a private 1-level vector context of n rows (created once, cached).
    The reference's vector-level entry points (``cgs2_orthogonalize`` and
    friends) take bare arrays; this is where their device work runs."""
    import weakref
    for ref in reversed(_LIVE):
        c = ref()
        if c is not None and c.h is not None and c.device == device and c.nranks == nranks \
                and c.level_info(0)["n"] == n:
            return c
    if nranks != 1:
        raise RuntimeError(f"no live {nranks}-rank context with {n} rows: build the hierarchy first")
    from .geometry import GlobalProblem
    ctx = Context(GlobalProblem.from_local(n, 1, 1, 1).domain(0), 1)
    _VECTOR_CTX.append(ctx)  # keep it alive for later calls
    return ctx


_VECTOR_CTX = []


class Context:
    def __init__(self, domain, levels, nu1=1, nu2=1, nu_c=1, world=None):
        rt = runtime()
        self.device = rt.device
        self.stream = rt.stream
        self.nranks = 1 if world is None else world.nranks
        self.rank = domain.rank
        self.levels = levels
        import os
        uid = None
        # HPG_NCCL=0: no NCCL communicator, peer memory only (ranks may share a GPU)
        self.nccl = self.nranks > 1 and os.environ.get("HPG_NCCL", "1") != "0"
        if self.nccl:
            uid = C.create_string_buffer(world.nccl_uid(), 128)
        h = C.c_void_p()
        L = _lib.lib()
        _lib.check(L.hpg_create(C.byref(h), rt.device.index, domain.rank, self.nranks,
                                _lib.ints(*domain.proc_dims), _lib.ints(*domain.local_dims),
                                levels, nu1, nu2, nu_c, uid, C.c_void_p(rt.stream_ptr)))
        self.h = h
        self._info = [self._level_info(l) for l in range(levels)]
        self.p2p = False
        if self.nranks > 1:
            self._open_peer_memory(world)
        import weakref
        _LIVE[:] = [r for r in _LIVE if r() is not None]
        _LIVE.append(weakref.ref(self))

    def _open_peer_memory(self, world):
        """Map every rank's symmetric buffer (CUDA IPC over NVLink); NCCL stays as
        the fallback data path when peer access is unavailable."""
        import os
        if os.environ.get("HPG_P2P", "1") == "0":
            if not self.nccl:
                raise RuntimeError("HPG_P2P=0 with HPG_NCCL=0 leaves no data path")
            return
        buf = C.create_string_buffer(64)
        self.call("hpg_p2p_handle", buf, 64)
        handles = world.gather(self.rank, bytes(buf.raw))
        handles = world.broadcast_bytes(handles)
        blob = C.create_string_buffer(b"".join(handles), 64 * self.nranks)
        rc = _lib.lib().hpg_p2p_open(self.h, blob, 64)
        ok = world.all_reduce_sum(self.rank, 1 if rc == 0 else 0) == self.nranks
        if not ok:
            if not self.nccl:
                raise RuntimeError("peer memory unavailable and HPG_NCCL=0: no data path")
            self.set_option("p2p", 0)
        world.barrier()
        self.p2p = ok

    def call(self, name, *args):
        if self.h is None:
            raise RuntimeError("context already destroyed")
        _lib.check(getattr(_lib.lib(), name)(self.h, *args))

    def _level_info(self, l):
        buf = np.zeros(len(INFO_KEYS), dtype=np.int64)
        self.call("hpg_level_info", l, buf.ctypes.data_as(C.POINTER(C.c_int64)), len(INFO_KEYS))
        return dict(zip(INFO_KEYS, (int(v) for v in buf)))

    def level_info(self, l):
        return self._info[l]

    def launches(self):
        return int(_lib.lib().hpg_launch_count(self.h))

    def timers(self, mode, seconds=None):
        out = np.zeros(8) if seconds is None else seconds
        self.call("hpg_timers", mode, out.ctypes.data_as(C.POINTER(C.c_double)))
        if mode in (0, 1):
            self.timing = mode == 1
        return out

    def set_option(self, key, value):
        self.call("hpg_set_option", key.encode(), int(value))
        self.__dict__.setdefault("_opts", {})[key] = int(value)

    def option(self, key):
        """Current value of a boolean library option (set here, else HPG_<KEY>, else the default)."""
        opts = self.__dict__.get("_opts", {})
        if key in opts:
            return opts[key]
        env = os.environ.get("HPG_" + key.upper())
        return BOOL_DEFAULTS[key] if env is None else int(env[:1] != "0")

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
