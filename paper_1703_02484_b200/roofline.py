"""Algorithmic-byte accounting of the O(N) step (host side, for reporting).

The persistent step kernels run many short memory-bound passes (integrate,
pass-through check, flag passes, independent-set rounds, flips, overlap
sweeps, incidence builds, Verlet rebuilds, short-range forces).  Each step
reports how many of each it ran (bd_stats_t.work[], csrc/bd_step.cuh WK_*);
this module turns the counts into the minimum bytes those passes must move
(per-unit figures of SURVEY.md §8(d), N particles, E = 3N edges, F = 2N
triangles, P stored pairs), so that bytes / step time is the achieved
bandwidth to compare with the HBM roofline.
"""

from __future__ import annotations

# bytes per pass -- SURVEY.md §8(d); n particles, e edges, t triangles,
# p Verlet pairs (short-range force / list build), q overlap pairs (the
# triangulation edges, or the Verlet overlap candidates without a triangulation)
PASS_BYTES = {
    "integrate": lambda n, e, t, p, q: 64 * n,                     # r pos, r F, w prev, w pos
    "apply_crossings": lambda n, e, t, p, q: 30 * t + 2 * n,       # tri_v + shifts r/w, crossings
    "edge_inversion": lambda n, e, t, p, q: 8 * e + 32 * n,        # edge_v + prev/cur positions
    "flag_pass": lambda n, e, t, p, q: 11 * e + 18 * t + 16 * n,   # edge quad gather + flag write
    "flag_edges_wl": lambda n, e, t, p, q: 11 + 36 + 32 + 8,       # per re-evaluated edge: quad, 4 positions, list
    "area_pass": lambda n, e, t, p, q: 19 * t + 16 * n,            # tri_v, shifts, positions, flag
    "lfmis_round": lambda n, e, t, p, q: 17 * e,                   # status of the edge + 4 neighbours
    "flips": lambda n, e, t, p, q: 190,                            # per flipped edge
    "overlap_pass": lambda n, e, t, p, q: 8 * q + 32 * n,          # pair list + positions
    "overlap_apply": lambda n, e, t, p, q: 25 * q + 32 * n,        # incidence, contributions, positions r/w
    "incidence": lambda n, e, t, p, q: 24 * q,                     # CSR of pairs per particle
    "verlet_rebuild": lambda n, e, t, p, q: 16 * n + 8 * p,
    "sr_force": lambda n, e, t, p, q: 8 * p + 40 * n,
}


def step_bytes(work: dict, n: int, ne: int, nt: int, pairs: int = 0, overlap_pairs: int | None = None) -> int:
    """Algorithmic bytes of one step from its work counters."""
    q = ne if overlap_pairs is None else overlap_pairs
    return int(sum(PASS_BYTES[k](n, ne, nt, pairs, q) * int(v) for k, v in work.items() if k in PASS_BYTES))


def hbm_peak_gbs(measured: dict, default: float = 6538.6) -> float:
    """HBM copy bandwidth from MEASURED_PEAKS.json (driver-written), else the recipe's figure."""
    for key in ("hbm_gbs", "hbm_copy_gbs", "hbm_burst_gbs", "hbm_GBps"):
        if key in measured:
            try:
                return float(measured[key])
            except (TypeError, ValueError):
                pass
    return default


PHASES = {  # pass kinds timed together (bd_stats_t.work timers)
    "maintenance": (("edge_inversion", "flag_pass", "flag_edges_wl", "area_pass", "lfmis_round", "flips"),
                    "t_maintain_ns"),
    "overlap": (("overlap_pass", "overlap_apply", "apply_crossings"), "t_overlap_ns"),
    "incidence": (("incidence",), "t_incidence_ns"),
    "verlet": (("verlet_rebuild",), "t_verlet_ns"),
    "sr_force": (("sr_force",), "t_sr_force_ns"),
    "pre": ((), "t_pre_ns"),
    "integrate": (("integrate",), "t_integrate_ns"),
}


def phase_breakdown(work: dict) -> dict:
    """Share of the step kernel's time per phase group (device clock of the leader thread)."""
    tot = max(int(work.get("t_total_ns", 0)), 1)
    # the SR force and the Verlet rebuild it triggers run inside "pre" in the triangulation driver
    out = {name: work.get(t, 0) / tot for name, (_, t) in PHASES.items() if name != "pre"}
    out["pre"] = max(0.0, work.get("t_pre_ns", 0) - work.get("t_sr_force_ns", 0) - work.get("t_verlet_ns", 0)) / tot
    out["other"] = max(0.0, 1.0 - sum(out.values()))
    return out


def phase_roofline(work: dict, n: int, ne: int, nt: int, pairs: int = 0, overlap_pairs: int | None = None) -> dict:
    """Achieved algorithmic bandwidth per phase group: {name: (bytes, ns, GB/s)}."""
    q = ne if overlap_pairs is None else overlap_pairs
    out = {}
    for name, (kinds, t) in PHASES.items():
        b = sum(PASS_BYTES[k](n, ne, nt, pairs, q) * work.get(k, 0) for k in kinds)
        ns = work.get(t, 0)
        if ns > 0:
            out[name] = {"bytes": float(b), "ns": float(ns), "GBs": float(b / ns)}
    return out
