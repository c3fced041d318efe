"""Snapshot / locality-flag / per-step CSV files (paper_1703_02484_b200/io.py)
against files the reference wrote (tests/golden/make_golden_io.py):
byte-identical output, exact round trips, the reference's error messages."""

import os
import types as _types

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "io")


def inputs():
    z = np.load(os.path.join(GOLD, "inputs.npz"))
    return {k: z[k] for k in z.files}


def fake_system(pos, types, L):
    from paper_1703_02484_b200.core import PeriodicBox
    return _types.SimpleNamespace(positions=pos, type_of=types, n=pos.shape[0], box=PeriodicBox(float(L)))


def series(z):
    from paper_1703_02484_b200.dynamics import StepStats
    cols = [str(c) for c in z["cols"]]
    ints = {"step", "overlap_iterations", "flip_passes", "inversion_repairs", "rollbacks"}
    return [StepStats(**{c: (int(v) if c in ints else float(v)) for c, v in zip(cols, row)}) for row in z["series"]]


def read(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return fh.read()


def test_snapshot_bytes_and_round_trip(tmp_path):
    from paper_1703_02484_b200 import io
    z = inputs()
    p = tmp_path / "s.txt"
    io.write_snapshot(fake_system(z["pos"], z["types"], z["L"]), float(z["t"]), str(p))
    assert p.read_bytes() == read("snapshot.txt")
    pos, typ, box, t = io.read_snapshot(os.path.join(GOLD, "snapshot.txt"))
    assert np.array_equal(pos, z["pos"]) and np.array_equal(typ, z["types"])
    assert box.length == float(z["L"]) and t == float(z["t"])


def test_flags_bytes_and_round_trip(tmp_path):
    from paper_1703_02484_b200 import io
    z = inputs()
    p = tmp_path / "f.txt"
    io.write_locality_flags(z["flags"], str(p))
    assert p.read_bytes() == read("flags.txt")
    assert np.array_equal(io.read_locality_flags(str(p)), z["flags"])


@pytest.mark.parametrize("name,cid,k", [("run.csv", "cfg-test", 14), ("run_short.csv", "short", 5)])
def test_csv_bytes_and_round_trip(tmp_path, name, cid, k):
    from paper_1703_02484_b200 import io
    z = inputs()
    rows = series(z)[:k]
    p = tmp_path / name
    io.write_csv(io.RunReport(cid, int(z["pos"].shape[0]), rows, warmup=10), str(p))
    assert p.read_bytes() == read(name)
    back, summary = io.read_csv(os.path.join(GOLD, name))
    assert [(s.step, s.dt_used, s.force_ms, s.overlap_iterations, s.rollbacks) for s in back] == \
        [(s.step, s.dt_used, s.force_ms, s.overlap_iterations, s.rollbacks) for s in rows]
    if k > 10:
        assert summary == {key: v for key, v in io.aggregate(rows, 10).items() if key != "steps"}
    else:
        assert summary == {}


def test_reader_errors(tmp_path):
    from paper_1703_02484_b200 import io
    from paper_1703_02484_b200.core import BrownsimError, ConfigError
    bad = tmp_path / "bad.txt"
    bad.write_text("# not-a-snapshot\n")
    with pytest.raises(BrownsimError, match=":1: not a brownsim snapshot header"):
        io.read_snapshot(str(bad))
    bad.write_text("# brownsim-snapshot v1 N=3 L=2 t=0\n0 0 0\n")
    with pytest.raises(BrownsimError, match="truncated file, missing particle row 1"):
        io.read_snapshot(str(bad))
    bad.write_text("# brownsim-snapshot v1 N=1 L=2 t=0\n0 0\n")
    with pytest.raises(BrownsimError, match=":2: expected 'x y type'"):
        io.read_snapshot(str(bad))
    bad.write_text("# brownsim-snapshot v1 N=1 L=2 t=0\n0 0 0\n1 1 1\n")
    with pytest.raises(BrownsimError, match="more rows follow"):
        io.read_snapshot(str(bad))
    bad.write_text("step,nope\n")
    with pytest.raises(BrownsimError, match="unexpected header"):
        io.read_csv(str(bad))
    with pytest.raises(ConfigError):
        io.aggregate(series(inputs())[:3], 3)


@pytest.mark.gpu
def test_snapshot_of_a_device_simulation(tmp_path):
    """A snapshot of a running simulation restores its exact positions."""
    import sys
    sys.path.insert(0, HERE)
    from golden_io import load
    from helpers import product_sim
    from paper_1703_02484_b200 import io
    sim = product_sim(load("lr_c0_n256"))
    sim.run(3)
    p = tmp_path / "snap.txt"
    io.write_snapshot(sim.sys, 0.03, str(p))
    pos, typ, box, t = io.read_snapshot(str(p))
    assert np.array_equal(pos, sim.sys.positions) and box.length == sim.sys.box.length and t == 0.03
    rep = io.RunReport("lr_c0_n256", 256, sim.run(12), warmup=10)
    io.write_csv(rep, str(tmp_path / "r.csv"))
    back, summary = io.read_csv(str(tmp_path / "r.csv"))
    assert [s.flip_passes for s in back] == [s.flip_passes for s in rep.series] and summary
