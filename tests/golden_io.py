"""Shared loaders for the golden fixtures (tests/golden/*.npz, made by make_golden.py)."""

from __future__ import annotations

import hashlib
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TRI_KEYS = ("tri_v", "tri_shift", "tri_edge", "edge_v", "edge_tri", "edge_opp")
STAT_KEYS = ("dt_used", "overlap_iterations", "flip_passes", "inversion_repairs", "rollbacks",
             "n_overlapping")
SCENARIOS = ("lr_c0_n256", "lr_c3_n512", "lr_rollback_n64", "sr_tri_n512", "lrsr_tri_n256",
             "sr_verlet_n512", "cfg1_lr_c0_n1024")


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def init_tri(rec: dict) -> dict:
    return {k: rec["init_" + k] for k in TRI_KEYS}


def final_tri(rec: dict) -> dict:
    return {k: rec["final_" + k] for k in TRI_KEYS}


def tri_hash(arrays: dict) -> str:
    h = hashlib.sha256()
    for k in TRI_KEYS:
        h.update(np.ascontiguousarray(arrays[k]).tobytes())
    return h.hexdigest()


def pos_hash(pos) -> str:
    return hashlib.sha256(np.ascontiguousarray(pos, np.float64).tobytes()).hexdigest()
