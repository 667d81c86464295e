"""N>1 host logic on CPU: two processes over gloo (the GPU path uses the same
World for bootstrap and control, NCCL for data).  Checks the rank-ordered
reduction (ref: comm.py:97-108), gather/broadcast, the NCCL unique-id
bootstrap, and that neighbouring ranks' halo plans mirror each other
(send list of r->q == halo slice of q<-r, ref: comm.py:180-236)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world_size, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world_size), LOCAL_RANK=str(rank))
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2507_11512_b200.comm import World
    from paper_2507_11512_b200.geometry import GlobalProblem
    from paper_2507_11512_b200.problem import host_level
    from paper_2507_11512_b200.comm import HaloPlan
    out = {}
    try:
        w = World(world_size)
        assert w.rank == rank
        vals = np.array([0.1 * (rank + 1), 1e16 * (-1) ** rank, 1.0], dtype=np.float32)
        s = w.all_reduce_sum(rank, vals)
        ref = vals * 0
        parts = [np.array([0.1 * (r + 1), 1e16 * (-1) ** r, 1.0], dtype=np.float32) for r in range(world_size)]
        acc = parts[0].copy()
        for p in parts[1:]:
            acc = acc + p
        out["allreduce_ordered"] = bool(np.array_equal(s, acc)) and s.dtype == ref.dtype
        g = w.gather(rank, rank * 10)
        out["gather"] = g == [10 * r for r in range(world_size)] if rank == 0 else g is None
        out["runs"] = w.run(lambda world, r: r + 100) == [100 + r for r in range(world_size)]
        uid = w.nccl_uid()
        allu = w.gather(rank, uid)
        out["uid"] = (len(uid) == 128 and len(set(allu)) == 1) if rank == 0 else len(uid) == 128
        # validation sub-world of the first k ranks (ref: bench.py:165-167)
        k = world_size - 1
        sub = w.subworld(k)
        if rank < k:
            out["subworld"] = (sub.nranks == k and sub.all_reduce_sum(rank, rank + 1) == k * (k + 1) // 2
                               and sub.run(lambda world, r: r) == list(range(k)))
        else:
            out["subworld"] = sub is None
        w.barrier()
        # default factor_ranks grid, and x-axis splits through the process-grid override
        grids = [None, (world_size, 1, 1)] + ([(2, 2, 1), (2, 1, 2)] if world_size == 4 else [])
        for gi, dims in enumerate(grids):
            gp = GlobalProblem.from_local(4, 4, 4, world_size, proc_dims=dims)
            d = gp.domain(rank)
            plan = HaloPlan.__new__(HaloPlan)
            plan.domain = d
            sends = {nb: len(v) for nb, v in plan.send_rows().items()}
            _, cols, _, _, meta = host_level(d.local_dims, d.coords, d.proc_dims)
            everyone = w.gather(rank, (sends, meta["halo"]))
            if rank == 0:
                # total sent to rank q by all peers == q's halo size
                for q_ in range(world_size):
                    got = sum(everyone[r][0].get(q_, 0) for r in range(world_size))
                    out[f"mirror_{gi}_{q_}"] = got == everyone[q_][1] and got > 0
    except Exception as e:  # report, do not hang the parent
        out["error"] = repr(e)
    q.put((rank, out))


@pytest.mark.parametrize("world_size", [2, 4])
def test_world_over_gloo(world_size):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world_size, port, q)) for r in range(world_size)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, out in res.items():
        assert "error" not in out, out
        assert out["allreduce_ordered"] and out["gather"] and out["runs"] and out["uid"], out
        assert out["subworld"], out
    for k, v in res[0].items():
        if k.startswith("mirror_"):
            assert v, (k, res)
