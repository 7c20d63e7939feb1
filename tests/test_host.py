"""Host-side logic of the drop-in surface (CPU only): mesh layout/init,
stencil tables vs the oracle, colour ids, dispatch errors, config, CSV."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_1810_04033_b200 as sl
from oracle import restate as R
from paper_1810_04033_b200 import _native, runner, strategies

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_flat_index_formula():
    m = sl.Mesh(2, 5)
    assert m.flat_index((1, 1)) == 8 and m.flat_index((6, 6)) == 48
    m3 = sl.Mesh(3, 3)
    assert m3.flat_index((1, 2, 3)) == (3 * 5 + 2) * 5 + 1
    for bad in ((7, 0), (0, -1), (1,)):
        with pytest.raises(IndexError):
            m.flat_index(bad)
    assert m.coord_of(m.flat_index((3, 4))) == (3, 4)


def test_constructor_rejects_bad_shapes():
    for dim, n in ((1, 4), (4, 4), (2, 0)):
        with pytest.raises(ValueError):
            sl.Mesh(dim, n)


def test_init_matches_reference_digests():
    with open(os.path.join(GOLDEN, "reference_digests.json")) as fh:
        want = json.load(fh)["init"]
    for key, digest in want.items():
        dim, n, seed, b = key.split("/")
        m = sl.make_mesh(int(dim), int(n), seed=int(seed), boundary_value=float(b))
        assert hashlib.sha256(m.values.tobytes()).hexdigest() == digest


def test_rhs_init_matches_oracle():
    m = sl.Mesh(3, 5)
    sl.init_rhs(m, 43)
    assert np.array_equal(m._rhs_host, R.init_f(3, 5, 43).ravel())
    assert m.omega == 0.8 and m.has_rhs


def test_stencil_tables_equal_oracle_restatement():
    for name, kind in sl.STENCILS.items():
        dim, offs, w, wc, c = R.STENCIL_TABLE[name]
        assert (kind.dim, kind.offsets, kind.weights, kind.centre_weight, kind.colours) == (dim, offs, w, wc, c)


def test_colour_of_matches_reference_examples():
    assert sl.colour_of(sl.FD5, (1, 1)) == 0 and sl.colour_of(sl.FD5, (2, 1)) == 1
    assert sl.colour_of(sl.FE9, (2, 2)) == 3
    assert sl.colour_of(sl.FE27, (2, 1, 2)) == 5
    for name, kind in sl.STENCILS.items():
        coords = [(3, 4), (1, 2)] if kind.dim == 2 else [(3, 4, 5), (2, 2, 1)]
        for c in coords:
            assert sl.colour_of(kind, c) == R.colour_of(name, c)


def test_same_colour_never_adjacent():
    import itertools
    for kind in sl.STENCILS.values():
        n = 5 if kind.dim == 2 else 4
        mesh = sl.Mesh(kind.dim, n)
        by = {}
        for c in mesh.interior_coords():
            by.setdefault(sl.colour_of(kind, c), []).append(c)
        for cells in by.values():
            for a, b in itertools.combinations(cells, 2):
                assert not kind.is_adjacent(a, b)


def test_plan_colour_partition():
    plan = sl.SweepPlan(sl.Mesh(2, 5), sl.FD5, sl.CostModel())
    assert [len(c) for c in plan.colour_cells] == [13, 12]
    first = sl.Mesh(2, 4).flat_index((1, 1))
    assert sl.SweepPlan(sl.Mesh(2, 4), sl.FE9, sl.CostModel()).colour_cells[0][0] == first


def test_dispatch_errors_follow_reference():
    m = sl.Mesh(2, 4)
    with pytest.raises(ValueError):
        sl.run_sweep("bogus", m, sl.FD5, sl.CostModel())
    with pytest.raises(ValueError):
        sl.run_sweep("colouring", m, sl.FD5, sl.CostModel(), pool=None)
    with pytest.raises(NotImplementedError):
        sl.run_sweep("nd", m, sl.FD5, sl.CostModel(), pool=sl.DevicePool())
    assert strategies.canonical_strategy("hyb_sync") == "hyb-sync"
    with pytest.raises(ValueError):
        sl.SweepPlan(sl.Mesh(3, 4), sl.FD5, sl.CostModel())


def test_cost_model_descriptor():
    assert sl.CostModel("const", 0).is_free
    assert not sl.CostModel("const", 3).is_free and not sl.CostModel("ramp").is_free
    d = sl.CostModel("const", 3).descriptor()
    assert (d.mode, d.k) == (_native.SL_COST_CONST, 3)
    assert sl.CostModel("ramp").descriptor().mode == _native.SL_COST_RAMP
    assert sl.CostModel("ramp").k_for_rank(99, 100) == 99
    with pytest.raises(ValueError):
        sl.CostModel("const", -1)


def test_stencil_kind_accepts_zero_weights_rejects_positive():
    with pytest.raises(AssertionError):
        sl.StencilKind("bad", 2, ((0, -1), (0, 1)), (1.0, -1.0), 0.0, 2)
    assert sl.FE27Q1.weights.count(0.0) == 6


def test_bench_config_validation():
    runner.BenchConfig(dim=2, stencil="fe9", strategy="hyb-sync").validated()
    for bad in (dict(dim=4), dict(stencil="nope"), dict(dim=3, stencil="fd5"),
                dict(strategy="nd"), dict(sizes=(0,)), dict(sweeps=0), dict(reps=0)):
        with pytest.raises(runner.ConfigError):
            runner.BenchConfig(**bad).validated()
    assert runner.parse_cost("const:7").k == 7
    with pytest.raises(runner.ConfigError):
        runner.parse_cost("linear")


def test_csv_round_trip():
    r = runner.BenchResult(2, 16, "fd5", "const:0", "colouring", 1, "static", 1, 10,
                           [0.5, 0.25], ["a", "a"])
    rows = runner.format_csv_rows([r])
    assert rows[0] == runner.CSV_HEADER
    back = runner.parse_csv("\n".join(rows))
    assert back[0].seconds == [0.5, 0.25] and back[0].digests == ["a", "a"]
    assert rows[1].endswith(",a,,1") and back[0].gpus == 1
    # reference-layout CSV (no device columns) still parses
    ref = [runner.REFERENCE_CSV_HEADER] + [",".join(row.split(",")[:13]) for row in rows[1:]]
    back = runner.parse_csv(ref)
    assert back[0].seconds == [0.5, 0.25]
    with pytest.raises(ValueError):
        runner.parse_csv([runner.CSV_HEADER, "1,2,3"])


def test_cli_configuration_errors_exit_2(capsys):
    from paper_1810_04033_b200 import cli
    assert cli.main(["run", "--dim", "3", "--stencil", "fd5"]) == 2
    assert cli.main(["run", "--cost", "linear"]) == 2
    assert cli.main(["run", "--strategy", "nd"]) == 2
    assert cli.main(["trace"]) == 2
    assert cli.main(["verify", "--suite", "races"]) == 2
    assert "configuration error" in capsys.readouterr().err


def test_schedule_parse():
    assert sl.Schedule.parse("dynamic:4").describe() == "dynamic:4"
    assert sl.Schedule.parse("static").describe() == "static"
    with pytest.raises(ValueError):
        sl.Schedule("guided")


def test_device_entry_points_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_1810_04033_b200._native import NativeLibraryError
    m = sl.make_mesh(2, 4, seed=1)
    with pytest.raises(NativeLibraryError):
        sl.run_sweep("colouring", m, sl.FD5, sl.CostModel(), pool=sl.DevicePool())


def test_stencil_lab_import_name_reaches_the_gpu_package():
    """`import stencil_lab` is the reference's import name (reference
    __init__.py:8-27); its modules are this package's."""
    import stencil_lab
    import stencil_lab.bench
    import stencil_lab.kernels
    import stencil_lab.mesh
    import stencil_lab.strategies
    from stencil_lab.taskrt import Schedule
    assert stencil_lab.strategies is strategies
    assert stencil_lab.bench.StrategyRunner is runner.StrategyRunner
    assert stencil_lab.sweep_colouring is sl.sweep_colouring
    assert stencil_lab.make_mesh is sl.make_mesh
    assert Schedule is sl.Schedule
    with pytest.raises(ImportError, match="nested dissection"):
        from stencil_lab import dissect  # noqa: F401


def test_read_values_is_read_only_and_keeps_the_device_authoritative():
    """`values` hands out a writable view (reference semantics) and therefore
    marks the host copy authoritative; `read_values` must not."""
    class HostOnly(type(sl.make_mesh(2, 6, seed=5))):
        __slots__ = ()

        def _dev_to_host(self):           # no GPU here: the "download" is a no-op
            pass

    m = HostOnly(2, 6)
    sl.init(m, 5)
    m._where = "dev"                      # as after a device sweep
    v = m.read_values()
    assert m._where == "dev"
    assert not v.flags.writeable
    with pytest.raises(ValueError):
        v[0] = 1.0
    assert np.array_equal(v, m._host)
    m.values[0] = 2.0                     # the writable accessor flips the state
    assert m._where == "host" and m._host[0] == 2.0
