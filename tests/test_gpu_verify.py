"""Device verification suites and the CLI (reference bench.py:285-522,
cli.py; tests/test_bench.py:134-153, tests/test_acceptance.py:133-138)."""

import json
import os

import pytest

import paper_1810_04033_b200 as sl
from paper_1810_04033_b200 import cli, runner

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_serial_budget_equals_reference():
    with open(os.path.join(GOLDEN, "reference_digests.json")) as fh:
        want = json.load(fh)["convergence"]
    for key, budget in want.items():
        name = key.split("/")[0]
        n = int(key.split("n=")[1].split("/")[0])
        assert sl.serial_convergence_budget(name, n, seed=7) == budget, key


def test_verify_oracle_passes():
    report = sl.verify_oracle(threads=(2,), n2=6, n3=4, sweeps=2)
    assert report.ok, report.lines
    assert all(ln.endswith("bit-equal") for ln in report.lines)


def test_criterion_06_convergence_within_twice_serial_budget():
    report = sl.verify_convergence(threads=2, cases=(("fd5", 33), ("fd7", 17)))
    assert report.ok, report.lines
    assert len(report.lines) == 2 * (1 + len(sl.GPU_STRATEGIES))


def test_cli_verify_and_run(tmp_path, capsys):
    assert cli.main(["verify", "--suite", "oracle"]) == 0
    assert "verify oracle: PASS" in capsys.readouterr().out
    out = tmp_path / "r.csv"
    assert cli.main(["run", "--size", "8,33", "--stencil", "fe9", "--strategy", "colouring",
                     "--sweeps", "100", "--reps", "2", "--csv", str(out)]) == 0
    rows = out.read_text().splitlines()
    assert rows[0] == runner.CSV_HEADER
    for r in runner.parse_csv(rows):
        assert r.common_digest() != "mixed"      # every repetition bit-identical
        assert r.gpus == 1 and r.device
    assert cli.main(["run", "--size", "8", "--strategy", "serial", "--sweeps", "3",
                     "--reps", "1"]) == 0


def test_cost_run_through_benchmark():
    (r,) = sl.run_benchmark(sl.BenchConfig(sizes=(16,), stencil="fd5", strategy="colouring",
                                           cost=sl.CostModel("const", 5), sweeps=3, reps=1))
    (r0,) = sl.run_benchmark(sl.BenchConfig(sizes=(16,), stencil="fd5", strategy="colouring",
                                            sweeps=3, reps=1))
    assert r.digests == r0.digests
