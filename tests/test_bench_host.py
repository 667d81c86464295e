"""Host logic of the benchmark driver (ref: tests/test_bench.py): configuration
validation, CLI exit codes, MatrixMarket dump -- no GPU needed."""
import json

import pytest

from paper_2507_11512_b200 import bench
from paper_2507_11512_b200.bench import BenchConfig, ConfigError, ValidationError, dump_matrix, main
from paper_2507_11512_b200.comm import ProtocolError


def test_default_config_is_valid():
    BenchConfig().validate()


@pytest.mark.parametrize("overrides", [
    {"local_nx": 12}, {"local_ny": 20}, {"local_nz": 4}, {"local_nx": 0}, {"local_nx": -8},
    {"ranks": 0}, {"validation_ranks": 0}, {"validation_ranks": 2}, {"restart": 0},
    {"tol": 0.0}, {"tol": -1e-9}, {"max_iters": 0}, {"nd_cap": 0}, {"time_seconds": -1.0},
    {"validation_mode": "turbo"}, {"coloring": "rainbow"}, {"nu1": 0}, {"nu2": 0}, {"nu_c": 0},
    {"mg_levels": 0},
])
def test_invalid_configs_rejected(overrides):
    # ref: tests/test_bench.py:35-60 (the same 20 cases)
    with pytest.raises(ConfigError):
        BenchConfig(**overrides).validate()


def test_shallow_hierarchy_relaxes_divisibility():
    BenchConfig(local_nx=12, local_ny=12, local_nz=12, mg_levels=3).validate()


def _cli(*extra):
    return ["--local-nx", "8", "--local-ny", "8", "--local-nz", "8", "--time-seconds", "0", *extra]


def test_cli_rejects_bad_geometry(capsys):
    assert main(["--local-nx", "12", "--local-ny", "8", "--local-nz", "8"]) == 2
    assert "configuration error" in capsys.readouterr().err


def test_cli_validation_failure_exit_code(monkeypatch, capsys):
    def boom(cfg):
        raise ValidationError("reference solve stalled")

    monkeypatch.setattr(bench, "run_benchmark", boom)
    assert main(_cli()) == 3
    assert "validation failed" in capsys.readouterr().err


def test_cli_protocol_failure_exit_code(monkeypatch, capsys):
    def boom(cfg):
        raise ProtocolError("replicated state diverged")

    monkeypatch.setattr(bench, "run_benchmark", boom)
    assert main(_cli()) == 4
    assert "protocol error" in capsys.readouterr().err


def test_cli_unknown_flag_exits_two():
    with pytest.raises(SystemExit) as exc:
        main(["--frequency", "9000"])
    assert exc.value.code == 2


def test_cli_report_file(monkeypatch, tmp_path, capsys):
    fake = {"config": {}, "validation": {}, "mxp": {}, "double": {},
            "summary": {"penalized_gflops": 1.0, "penalty": 1.0, "speedup": 1.0, "reps": 1}}
    monkeypatch.setattr(bench, "run_benchmark", lambda cfg: fake)
    path = tmp_path / "report.json"
    assert main(_cli("--report-path", str(path))) == 0
    assert json.loads(path.read_text())["summary"]["reps"] == 1
    out = capsys.readouterr().out
    assert "penalized" in out and str(path) in out


def test_dump_matrix(tmp_path):
    # ref: tests/test_bench.py:220-227 -> 8^3: 512 rows, 10,648 nnz
    path = tmp_path / "stencil.mtx"
    dump_matrix(BenchConfig(local_nx=8, local_ny=8, local_nz=8), str(path))
    lines = path.read_text().splitlines()
    assert lines[0].startswith("%%MatrixMarket")
    assert lines[1].split() == ["512", "512", "10648"]
    assert len(lines) == 2 + 10648
    # natural order, 1-based global ids, ascending columns within a row
    first = [tuple(map(float, l.split())) for l in lines[2:10]]
    assert first[0] == (1.0, 1.0, 26.0) and first[1] == (1.0, 2.0, -1.0)


@pytest.mark.parametrize("name,cfg", [
    ("l8r1", dict(local_nx=8, local_ny=8, local_nz=8)),
    ("l4r2", dict(local_nx=4, local_ny=4, local_nz=4, ranks=2, mg_levels=2)),
    ("l4r8", dict(local_nx=4, local_ny=4, local_nz=4, ranks=8, mg_levels=2)),
])
def test_dump_matrix_byte_identical_to_reference(tmp_path, name, cfg):
    import hashlib
    from conftest import load_golden
    path = tmp_path / "m.mtx"
    dump_matrix(BenchConfig(**cfg), str(path))
    assert hashlib.sha256(path.read_bytes()).hexdigest() == load_golden("mtx_sha256.json")[name]
