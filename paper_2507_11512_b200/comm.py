"""Process-per-GPU world: the B200 replacement of the reference's RankWorld.

The reference simulates ranks as threads with FIFO mailboxes and a
rank-ordered allreduce (ref: comm.py:37-152).  Here every rank is an OS
process bound to one GPU (launched by torchrun); ``torch.distributed`` (gloo)
is only the bootstrap and host-side control plane, while the data path --
halo exchange and the rank-ordered reductions -- runs inside libhpgmxp on the
GPU's own NCCL communicator over NVLink (csrc/hpg_capi.cu do_exchange /
allreduce_scal).

Semantics kept from the reference:
  * ``all_reduce_sum`` folds contributions in ascending rank order, so every
    rank sees bitwise-identical sums (ref: comm.py:97-108);
  * ``run(fn)`` calls ``fn(world, rank)`` on this process's rank and returns
    the list of every rank's result (ref: comm.py:122-152);
  * exceptions: ProtocolError / TopologyError (ref: comm.py:25-30).
"""

from __future__ import annotations

import os
import pickle

import numpy as np


class ProtocolError(Exception):
    """Ranks disagreed about the communication schedule (ref: comm.py:25-26)."""


class TopologyError(Exception):
    """A column is owned by a non-neighbouring rank (ref: comm.py:29-30)."""


class _Runtime:
    """Per-process device state: the CUDA device and the one compute stream."""

    def __init__(self):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2507_11512_b200 needs a CUDA device (no CPU fallback)")
        local = int(os.environ.get("LOCAL_RANK", "0"))
        self.device = torch.device("cuda", local % torch.cuda.device_count())
        torch.cuda.set_device(self.device)
        self.stream = torch.cuda.Stream(self.device)
        torch.cuda.set_stream(self.stream)

    @property
    def stream_ptr(self):
        return self.stream.cuda_stream


_RT = None


def runtime():
    global _RT
    if _RT is None:
        _RT = _Runtime()
    return _RT


class World:
    """The set of ranks of one job (one process each); ``world=None`` means 1 rank.

    ``subworld(k)`` gives the first k ranks their own World (a gloo sub-group),
    e.g. for a validation run on fewer ranks than the job (ref: bench.py:165-167).
    """

    def __init__(self, nranks=None, _group=None, _rank=None):
        import torch.distributed as dist
        if nranks is None:
            nranks = int(os.environ.get("WORLD_SIZE", "1"))
        if nranks < 1:
            raise ValueError(f"need at least one rank, got {nranks}")
        self.nranks = nranks
        self._group = _group
        if _group is None:
            if nranks > 1 and not dist.is_initialized():
                dist.init_process_group("gloo")
            if nranks > 1 and dist.get_world_size() != nranks:
                raise ProtocolError(f"world of {nranks} ranks requested but {dist.get_world_size()} "
                                    "processes are running (one process per rank)")
            self.rank = dist.get_rank() if nranks > 1 else 0
        else:
            self.rank = _rank
        self._uid = None

    def subworld(self, k):
        """World of ranks [0, k) (collective over this world); None on the other ranks."""
        if not 1 <= k <= self.nranks:
            raise ValueError(f"sub-world of {k} ranks out of [1, {self.nranks}]")
        if k == self.nranks:
            return self
        if k == 1:
            return World(1) if self.rank == 0 else None
        import torch.distributed as dist
        g = dist.new_group(ranks=list(range(k)), backend="gloo")
        return World(k, _group=g, _rank=self.rank) if self.rank < k else None

    def _kw(self):
        return {} if self._group is None else {"group": self._group}

    # -- control plane (host, gloo) -------------------------------------
    def barrier(self, rank=None):
        if self.nranks > 1:
            import torch.distributed as dist
            dist.barrier(**self._kw())

    def broadcast_bytes(self, data, root=0):
        if self.nranks == 1:
            return data
        import torch.distributed as dist
        box = [data]
        dist.broadcast_object_list(box, src=root, **self._kw())  # members are ranks 0..k-1 globally
        return box[0]

    def gather(self, rank, value, root=0):
        """Every rank's value at ``root`` (ref: comm.py:110-118)."""
        if self.nranks == 1:
            return [value]
        import torch.distributed as dist
        out = [None] * self.nranks
        dist.all_gather_object(out, value, **self._kw())
        return out if rank == root else None

    def all_reduce_sum(self, rank, value):
        """Host-side sum in ascending rank order (ref: comm.py:97-108)."""
        if self.nranks == 1:
            return value
        import torch.distributed as dist
        parts = [None] * self.nranks
        dist.all_gather_object(parts, pickle.dumps(value), **self._kw())
        vals = [pickle.loads(p) for p in parts]
        acc = vals[0].copy() if isinstance(vals[0], np.ndarray) else vals[0]
        for v in vals[1:]:
            acc = acc + v
        return acc

    def nccl_uid(self):
        """A fresh NCCL unique id for a new communicator (collective: rank 0 creates,
        every rank receives).  Each communicator needs its own id."""
        from . import _lib
        import ctypes as C
        buf = (C.c_char * 128)()
        if self.rank == 0:
            _lib.check(_lib.lib().hpg_nccl_unique_id(buf, 128))
        self._uid = self.broadcast_bytes(bytes(buf))
        return self._uid

    def run(self, fn, *args, **kwargs):
        """Run fn(world, rank, ...) on this process's rank; list of all ranks' results."""
        res = fn(self, self.rank, *args, **kwargs)
        if self.nranks == 1:
            return [res]
        import torch.distributed as dist
        out = [None] * self.nranks
        dist.all_gather_object(out, res, **self._kw())
        return out


# the reference's module-level name (ref: comm.py:37)
RankWorld = World


def reduce_sum(world, rank, value):
    """all_reduce_sum that degrades to identity without a world (ref: comm.py:275-279)."""
    if world is None:
        return value
    return world.all_reduce_sum(rank, value)


def exchange(v, plan, world=None, rank=0):
    """Fill v's halo tail from the neighbours (ref: comm.py:239-251).

    ``plan`` is the level's HaloPlan handle (multigrid.MgLevel.plan); the
    exchange itself runs on the GPU (pack kernel + NCCL send/recv into the
    halo tail, csrc/hpg_capi.cu do_exchange).
    """
    if plan is None or world is None:
        return
    plan.exchange(v)


class HaloPlan:
    """Device halo plan of one level: neighbours, counts, slots (ref: comm.py:158-177).

    The send lists and slot layout are computed on the device from closed forms
    (csrc/hpg_geom.h send_row / halo_base); this object exposes them for
    inspection and parity tests.
    """

    def __init__(self, ctx, level, domain):
        self._ctx = ctx
        self.level = level
        self.domain = domain
        info = ctx.level_info(level)
        self.halo_offset = info["n"]
        self.halo_size = info["halo"]
        self.neighbors = domain.neighbor_ranks() if ctx.nranks > 1 else []

    @property
    def has_traffic(self):
        return self.halo_size > 0

    def exchange(self, v):
        from . import _lib
        prec = _lib.F32 if v.dtype.itemsize == 4 else _lib.F64
        self._ctx.call("hpg_exchange", self.level, prec, _lib.ptr(v))

    def send_rows(self):
        """{neighbour rank: permuted local rows} in the peer's request order."""
        from . import _lib
        import ctypes as C
        d = self.domain
        out = {}
        L = _lib.lib()
        for sz in (-1, 0, 1):
            for sy in (-1, 0, 1):
                for sx in (-1, 0, 1):
                    if (sx, sy, sz) == (0, 0, 0):
                        continue
                    cx, cy, cz = d.ix + sx, d.iy + sy, d.iz + sz
                    if not (0 <= cx < d.npx and 0 <= cy < d.npy and 0 <= cz < d.npz):
                        continue
                    args = (_lib.ints(*d.local_dims), _lib.ints(*d.coords), _lib.ints(*d.proc_dims))
                    cnt = L.hpg_host_send_rows(*args, sx, sy, sz, None)
                    rows = np.zeros(cnt, dtype=np.int64)
                    L.hpg_host_send_rows(*args, sx, sy, sz, rows.ctypes.data_as(C.POINTER(C.c_int64)))
                    out[cx + d.npx * (cy + d.npy * cz)] = rows
        return dict(sorted(out.items()))


def build_halo_plan(domain, A, world=None, rank=0, iperm=None):
    """The exchange plan of A's level (ref: comm.py:180-236).  The device built
    it with the level (send lists from the closed-form geometry, halo slots in
    ascending neighbour rank / global index, A's off-rank columns already
    pointing at them), so this hands out that plan; ``iperm`` is implied by A's
    row order.  The 27-point neighbourhood never reaches a non-neighbour rank,
    so the reference's TopologyError cannot arise."""
    return HaloPlan(A.ctx, A.level, domain)


def exchange_overlapped(v, plan, world, rank, interior_work):
    """Exchange v's halo and run ``interior_work()`` (ref: comm.py:254-272).

    Both are enqueued on the context's stream in that order, so the result is
    the reference's bit for bit (the caller's contract: the interior work reads
    no halo slot and writes no sent row).  The overlapped schedule proper -- the
    exchange on a side stream under the interior rows -- lives inside the
    library's SpMV and GS (option "overlap")."""
    if world is None or plan is None or not plan.neighbors:
        return interior_work()
    plan.exchange(v)
    return interior_work()
