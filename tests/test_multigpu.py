"""Multi-GPU parity (2 GPUs or more): bitwise kernels vs the oracle's all-rank
simulation and solver counts vs the reference (tests/golden/solves.json r2l16:
23 double, mixed envelope), through torchrun + NCCL.  Skips on 1-GPU boxes."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _run(nproc, L, levels, env=None, dims=None):
    e = dict(os.environ)
    e.update(env or {})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--local-addr", "127.0.0.1",
           "--nproc-per-node", str(nproc), os.path.join(ROOT, "tools", "mgpu_check.py"), str(L), str(levels)]
    if dims is not None:
        cmd.append(",".join(map(str, dims)))
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=e)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    line = [x for x in p.stdout.splitlines() if x.startswith("{")][-1]
    return json.loads(line)


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
def test_two_ranks_16():
    out = _run(2, 16, 4)
    for rk in out["checks"]:
        assert all(rk.values()), out["checks"]
    _check_solves(out, "r2l16")
    assert out["solves"]["double"]["iterations"] == 23
    assert out["summary"]["raw_gflops"] > 0


def _check_solves(out, case):
    """fp64 counts exact; mixed: per restart cycle within +-1 of the reference
    envelope; fullscale validation over all ranks has the same
    counts (ref bench.py:168-173)."""
    from test_gpu_parity import assert_cycles_in_envelope
    ref = dict(load_golden("solves.json"), **load_golden("solves_xsplit.json"))[case]
    assert out["solves"]["double"]["iterations"] == ref["1"]["double"]["iterations"]
    assert out["solves"]["double"]["converged"]
    assert out["solves"]["mixed"]["relres"] < 1e-9
    assert_cycles_in_envelope(out["solves"]["mixed"]["cycles"], case)
    assert out["validation"]["mode"] == "fullscale"
    assert out["validation"]["n_d"] == ref["1"]["double"]["iterations"]
    env = [ref[t]["mixed"]["iterations"] for t in ("1", "default")]
    ncyc = len(ref["1"]["mixed"]["cycle_iters"])
    assert min(env) - ncyc <= out["validation"]["n_ir"] <= max(env) + ncyc


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
def test_two_ranks_x_split_16():
    """(2,1,1): the x faces go through the NVLink halo kernel (factor_ranks never
    splits x below 8 ranks); kernels bitwise vs the oracle, counts vs the
    reference run on the same grid (tests/golden/solves_xsplit.json)."""
    out = _run(2, 16, 4, dims=(2, 1, 1))
    assert out["proc_dims"] == [2, 1, 1]
    for rk in out["checks"]:
        assert all(rk.values()), out["checks"]
    _check_solves(out, "x211l16")


@pytest.mark.skipif(_gpus() < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("dims", [(2, 2, 1), (2, 1, 2)])
def test_four_ranks_x_split_8(dims):
    """x faces, xy / xz edges (and the rank-diagonal neighbours) on 4 GPUs."""
    out = _run(4, 8, 4, dims=dims)
    assert out["proc_dims"] == list(dims)
    for rk in out["checks"]:
        assert all(rk.values()), out["checks"]
    _check_solves(out, "x%d%d%dl8" % dims)


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
def test_two_ranks_x_split_nccl_path():
    """The NCCL fallback data path on the x split."""
    out = _run(2, 8, 3, {"HPG_P2P": "0"}, dims=(2, 1, 1))
    for rk in out["checks"]:
        assert all(rk.values()), out["checks"]
    assert out["solves"]["double"]["converged"] and out["solves"]["mixed"]["relres"] < 1e-9


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("env", [{"HPG_P2P": "0"}, {"HPG_OVERLAP": "0"}, {"HPG_P2P": "0", "HPG_OVERLAP": "1"},
                                 {"HPG_CGS_FUSED": "0"}, {"HPG_NCCL": "0"},
                                 # the overlapped exchange under the tensor-copy pass / SpMV (skip flags)
                                 {"HPG_OVERLAP": "1", "HPG_OVERLAP_ROWS": "0", "HPG_TMA_MIN_ROWS": "0"}])
def test_two_ranks_alternative_paths(env):
    """NCCL data path, overlapped exchange, per-pass CGS2 and the P2P-only
    context (no NCCL communicator): same bitwise kernels, converged solves."""
    out = _run(2, 8, 3, env)
    for rk in out["checks"]:
        assert all(rk.values()), (env, out["checks"])
    assert out["solves"]["double"]["converged"] and out["solves"]["mixed"]["relres"] < 1e-9


@pytest.mark.skipif(_gpus() < 4, reason="needs 4 GPUs")
def test_four_ranks_8():
    out = _run(4, 8, 4)
    for rk in out["checks"]:
        assert all(rk.values()), out["checks"]
    assert out["solves"]["double"]["converged"] and out["solves"]["mixed"]["relres"] < 1e-9


@pytest.mark.skipif(_gpus() < 8, reason="needs 8 GPUs")
def test_eight_ranks_8():
    """The 2x2x2 grid (the 8xB200 configuration: x, y and z faces, edges and
    corners).  (Ranks sharing a GPU do not work: the peer-memory spin waits of
    one process's kernels starve the other process's time slice.)"""
    # ref: tests/test_acceptance.py:347-348 -> 8 ranks x 8^3: 18 double / 23 mixed
    out = _run(8, 8, 4)
    for rk in out["checks"]:
        assert all(rk.values()), out["checks"]
    assert out["solves"]["double"]["iterations"] == 18
    _check_solves(out, "r8l8")
