"""The CPU oracle (oracle/bd_oracle.c) pinned against the reference's own
outputs (tests/golden/*.npz, produced by running the reference with
tests/golden/make_golden.py) and against third-party known answers.

Bar: bit-exact everywhere (the oracle restates the reference expression by
expression, without contraction)."""

import ctypes

import numpy as np
import pytest

from golden_io import SCENARIOS, STAT_KEYS, init_tri, load, pos_hash, tri_hash
from helpers import oracle_sim, stats_row
from oracle import oracle as O
from oracle.noise_np import CounterNormals, log_portable, normal_pairs, philox4x64


def test_philox_core_matches_numpy_known_answers():
    """Philox4x64-10 == numpy's np.random.Philox (counter pre-increment)."""
    key = (12345, 7)
    for ctr in ([0, 0, 0, 0], [5, 3, 2, 1], [2**64 - 2, 17, 3, 9]):
        bg = np.random.Philox(key=np.array(key, dtype=np.uint64), counter=np.array(ctr, dtype=np.uint64))
        raw = bg.random_raw(4)
        nxt = list(ctr)
        nxt[0] += 1
        ours = philox4x64(*[np.array([x], np.uint64) for x in nxt], *key)
        assert [int(o[0]) for o in ours] == [int(r) for r in raw]
        out = np.zeros(4, np.uint64)
        O.lib().bdo_philox.argtypes = [ctypes.c_void_p] * 3
        c = np.array(nxt, np.uint64)
        k = np.array(key, np.uint64)
        O.lib().bdo_philox(c.ctypes.data, k.ctypes.data, out.ctypes.data)
        assert [int(o) for o in out] == [int(r) for r in raw]


def test_portable_log_accuracy_and_c_agreement():
    x = np.random.default_rng(0).uniform(2.0**-104, 1.0, 50000)
    ours = log_portable(x)
    ulp = np.abs(ours - np.log(x)) / np.spacing(np.abs(np.log(x)))
    assert ulp.max() <= 1.0
    L = O.lib()
    L.bdo_log_export.restype = ctypes.c_double
    L.bdo_log_export.argtypes = [ctypes.c_double]
    assert all(L.bdo_log_export(float(v)) == float(w) for v, w in zip(x[:3000], ours[:3000]))


def test_counter_normals_c_equals_numpy():
    n = 20001
    out = np.empty(n)
    L = O.lib()
    L.bdo_normals(3, 2, 11, 0, n, out.ctypes.data)
    assert np.array_equal(out, normal_pairs(3, 2, 11, (n + 1) // 2).reshape(-1)[:n])


def test_counter_normals_statistics():
    z = normal_pairs(1, 2, 0, 200000).reshape(-1)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
    # clamped second moment 0.99499 (tests/test_core.py:113-121 of the reference)
    assert abs(np.mean(np.clip(z, -3, 3) ** 2) - 0.99499) < 0.01


def test_counter_normals_known_answer():
    k = load("kernels")
    assert np.array_equal(CounterNormals(5, stream=2, call=3).normals((7, 2)), k["noise_5_2_3"])


def test_long_range_kernel_bitwise():
    k = load("kernels")
    out, err = O.long_range(k["lr_pos"], k["lr_alpha"], k["lr_mu"], float(k["lr_L"]))
    assert np.array_equal(out, k["lr_out"]) and np.array_equal(err, k["lr_err"])


def test_verlet_pairs_and_short_range_bitwise():
    k = load("kernels")
    pa, pb = O.verlet_pairs(k["sr_pos"], float(k["sr_L"]), 3.0)
    assert np.array_equal(pa, k["sr_pa"]) and np.array_equal(pb, k["sr_pb"])
    g = O.cell_grid(k["sr_pos"], float(k["sr_L"]), 3.0)
    assert g[0] == int(k["sr_ncx"]) and np.array_equal(g[1], k["sr_order"]) and np.array_equal(g[2], k["sr_cell_start"])
    out, err = O.short_range(k["sr_pos"], k["sr_alpha"], k["sr_mu"], pa, pb, float(k["sr_L"]), 2.5)
    assert np.array_equal(out, k["sr_out"]) and np.array_equal(err, k["sr_err"])


def test_brute_force_verlet_order():
    k = load("kernels")
    pa, pb = O.verlet_pairs(k["bf_pos"], float(k["bf_L"]), 3.0)
    assert np.array_equal(pa, k["bf_pa"]) and np.array_equal(pb, k["bf_pb"])


def test_overlap_pass_and_max_sq_disp_bitwise():
    k = load("kernels")
    d, f, c = O.overlap_pass(k["sr_pos"], k["sr_oa"], k["sr_ob"], float(k["sr_L"]), 1.0)
    assert np.array_equal(d, k["ov_disp"]) and np.array_equal(f, k["ov_flags"]) and c == int(k["ov_count"])
    assert O.max_sq_disp(k["msd_pos"], k["sr_pos"], float(k["sr_L"])) == float(k["msd_val"])


@pytest.mark.parametrize("name", SCENARIOS)
def test_step_trajectories_bitwise(name):
    rec = load(name)
    sim = oracle_sim(rec)
    for s in range(len(rec["pos_hash"])):
        st = sim.step()
        assert st["status"] == 0
        assert stats_row(st) == list(rec["stats"][s]), f"step {s}"
        assert pos_hash(sim.pos) == rec["pos_hash"][s], f"step {s}"
        if sim.tri is not None:
            assert tri_hash(sim.tri.arrays()) == rec["tri_hash"][s], f"step {s}"
    assert sim.call == int(rec["calls"][-1])


def test_build_restore_matches_reference_final_arrays():
    """Reference quotient arrays + the oracle's restore_delaunay == reference build_initial."""
    b = load("build")
    for tag in ("a", "b"):
        pos, L = b[f"{tag}_pos"], float(b[f"{tag}_L"])
        pre = {k: b[f"{tag}_pre_{k}"] for k in ("tri_v", "tri_shift", "tri_edge", "edge_v", "edge_tri", "edge_opp")}
        t = O.OracleTri.from_arrays(pre, pos.shape[0], L)
        t.restore_delaunay(pos)
        for k, v in t.arrays().items():
            assert np.array_equal(v, b[f"{tag}_fin_{k}"]), (tag, k)
