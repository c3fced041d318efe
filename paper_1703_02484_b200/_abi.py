"""ctypes mirror of include/bd_b200.h (structs, constants, prototypes)."""

from __future__ import annotations

import ctypes

c_i64, c_u64, c_d, c_vp, c_int = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int

BD_OK = 0
BD_ERR_SINGULAR = 1
BD_ERR_NONCONV = 2
BD_ERR_STEPFAIL = 4
BD_ERR_FLIP = 5
BD_ERR_CAPACITY = 6
BD_ERR_BUILD = 7

BD_FORCE_LR = 0
BD_FORCE_SR = 1
BD_FORCE_LRSR = 2

BD_LR_EXACT = 0
BD_LR_FAST = 1
BD_LR_FAST_SYM = 2


class BdTri(ctypes.Structure):
    _fields_ = [("nv", c_i64), ("ne", c_i64), ("nt", c_i64),
                ("tri_v", c_vp), ("tri_shift", c_vp), ("tri_edge", c_vp),
                ("edge_v", c_vp), ("edge_tri", c_vp), ("edge_opp", c_vp)]


class BdParams(ctypes.Structure):
    _fields_ = [("n", c_i64), ("L", c_d),
                ("sigma", c_d), ("dt", c_d), ("diffusion", c_d), ("cap", c_d), ("clamp", c_d),
                ("r_cut", c_d), ("skin", c_d), ("tol", c_d),
                ("max_overlap_iters", c_i64), ("max_rollbacks", c_i64),
                ("seed", c_u64), ("stream", c_u64),
                ("force_mode", c_i64), ("lr_precision", c_i64),
                ("mi_lo", c_d), ("mi_hi", c_d), ("r_list", c_d), ("ncx", c_i64),
                ("pair_capacity", c_i64),
                ("abp_speed", c_d), ("abp_rot_diffusion", c_d), ("abp_clamp_angle", c_i64)]


class BdStats(ctypes.Structure):
    _fields_ = [("dt_used", c_d), ("overlap_iterations", c_i64), ("flip_passes", c_i64),
                ("inversion_repairs", c_i64), ("rollbacks", c_i64), ("n_overlapping", c_i64),
                ("status", c_i64), ("err_i", c_i64), ("err_k", c_i64), ("rebuilds", c_i64),
                ("calls", c_i64), ("reserved", c_i64 * 5), ("work", c_i64 * 24)]


# bd_stats_t.work[] counters (csrc/bd_step.cuh WK_*)
WORK_KEYS = ("integrate", "apply_crossings", "edge_inversion", "flag_pass", "area_pass", "lfmis_round", "flips",
             "overlap_pass", "overlap_apply", "incidence", "verlet_rebuild", "sr_force",
             "t_maintain_ns", "t_overlap_ns", "t_incidence_ns", "t_total_ns", "t_verlet_ns", "t_sr_force_ns",
             "t_pre_ns", "t_integrate_ns", "flag_edges_wl")


STATS_WORDS = ctypes.sizeof(BdStats) // 8


class BdState(ctypes.Structure):
    _fields_ = [("pos", c_vp), ("prev", c_vp), ("force", c_vp), ("alpha", c_vp), ("mu", c_vp),
                ("force_err", c_vp), ("image", c_vp), ("overlap_flags", c_vp),
                ("tri", BdTri), ("tri_backup", BdTri), ("call", c_vp), ("stats", c_vp),
                ("pair_a", c_vp), ("pair_b", c_vp), ("vl_snap", c_vp), ("vl_meta", c_vp),
                ("work", c_vp), ("work_bytes", c_i64), ("angles", c_vp)]


_PROTOS = None


def _protos():
    P = ctypes.POINTER
    return {
        "bd_prepare_params": ([P(BdParams)], None),
        "bd_workspace_bytes": ([P(BdParams), c_i64, c_i64], c_i64),
        "bd_pairs_workspace_bytes": ([c_i64, c_d, c_d, c_i64], c_i64),
        "bd_long_range_workspace_bytes": ([c_i64], c_i64),
        "bd_long_range_workspace_bytes_for": ([c_i64, c_int], c_i64),
        "bd_long_range_forces": ([c_vp, c_vp, c_vp, c_i64, c_d, c_i64, c_i64, c_int, c_vp, c_vp, c_vp, c_vp], c_int),
        "bd_short_range_forces": ([c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_d, c_d, c_vp, c_vp, c_vp, c_vp],
                                  c_int),
        "bd_overlap_pass": ([c_vp, c_i64, c_vp, c_vp, c_i64, c_d, c_d, c_d, c_vp, c_vp, c_vp, c_vp, c_vp], c_int),
        "bd_max_sq_displacement": ([c_vp, c_vp, c_i64, c_d, c_vp, c_vp], c_int),
        "bd_verlet_build": ([c_vp, c_i64, c_d, c_d, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp], c_int),
        "bd_probe_fp64": ([c_i64, c_vp, c_vp, P(c_d)], c_int),
        "bd_probe_barrier": ([c_i64, c_int, c_int, c_int, c_vp, c_vp, P(c_d)], c_int),
        "bd_probe_exact_arith": ([c_u64, c_i64, c_vp, c_vp], c_int),
        "bd_brute_overlaps": ([c_vp, c_i64, c_d, c_d, c_vp, c_vp], c_int),
        "bd_normals": ([c_u64, c_u64, c_u64, c_u64, c_i64, c_vp, c_vp], c_int),
        "bd_force": ([P(BdState), P(BdParams), c_vp], c_int),
        "bd_force_prepare": ([P(BdState), P(BdParams), c_vp], c_int),
        "bd_force_slots": ([P(BdState), P(BdParams), c_i64, c_i64, c_vp, c_vp], c_int),
        "bd_force_finish": ([P(BdState), P(BdParams), c_vp, c_vp], c_int),
        "bd_force_sym_partial": ([P(BdState), P(BdParams), c_int, c_int, c_vp, c_vp], c_int),
        "bd_force_sym_finish": ([P(BdState), P(BdParams), c_vp, c_vp], c_int),
        "bd_maintain_tri": ([P(BdState), P(BdParams), c_vp, c_vp], c_int),
        "bd_step_tri": ([P(BdState), P(BdParams), c_vp], c_int),
        "bd_run_tri": ([P(BdState), P(BdParams), c_i64, c_vp, c_vp], c_int),
        "bd_step_verlet": ([P(BdState), P(BdParams), c_vp, c_vp], c_int),
        "bd_run_verlet": ([P(BdState), P(BdParams), c_i64, c_vp, c_vp], c_int),
        "bd_step_abp": ([P(BdState), P(BdParams), c_vp, c_vp], c_int),
        "bd_run_abp": ([P(BdState), P(BdParams), c_i64, c_vp, c_vp], c_int),
        "bd_tri_restore_delaunay": ([P(BdState), P(BdParams), c_vp, c_vp], c_int),
        "bd_clear_status": ([P(BdState), c_vp], c_int),
        "bd_tri_audit_geometry": ([P(BdState), P(BdParams), c_vp, c_vp], c_int),
        "bd_integrate": ([P(BdState), P(BdParams), c_d, c_vp, c_vp, c_vp], c_int),
        "bd_integrate_noise": ([P(BdState), P(BdParams), c_d, c_vp, c_vp, c_vp, c_vp], c_int),
        "bd_sym_shard": ([c_i64, c_int, c_int, c_vp], c_int),
        "bd_timing_enable": ([c_i64], c_int),
        "bd_timing_read": ([c_vp, c_i64], c_i64),
        "bd_tri_apply_crossings": ([P(BdState), P(BdParams), c_vp, c_vp], c_int),
        "bd_tri_edge_inversion": ([P(BdState), P(BdParams), c_vp, c_vp], c_int),
        "bd_tri_signed_area2": ([P(BdState), P(BdParams), c_vp, c_vp], c_int),
        "bd_tri_delaunay_flags": ([P(BdState), P(BdParams), c_vp, c_vp], c_int),
        "bd_tri_inverted_edge_flags": ([P(BdState), P(BdParams), c_vp, c_vp], c_int),
        "bd_tri_flip_edges": ([P(BdState), P(BdParams), c_vp, c_i64, c_vp, c_vp], c_int),
        "bd_tri_repair_inversions": ([P(BdState), P(BdParams), c_i64, c_int, c_vp, c_vp], c_int),
        "bd_tri_restore_delaunay_ex": ([P(BdState), P(BdParams), c_i64, c_vp, c_vp], c_int),
        "bd_overlap_correct": ([P(BdState), P(BdParams), c_i64, c_int, c_vp, c_vp], c_int),
        "bd_tri_copy": ([P(BdTri), P(BdTri), c_vp], c_int),
        "bd_tri_build_workspace_bytes": ([c_i64, c_d], c_i64),
        "bd_tri_build_initial": ([c_vp, c_i64, c_d, P(BdTri), c_vp, c_i64, c_vp, c_vp], c_int),
        "bd_build_info": ([], ctypes.c_char_p),
    }


def declare(lib):
    """Prototypes of the entry points of include/bd_b200.h present in `lib`."""
    for name, (args, res) in _protos().items():
        if hasattr(lib, name):
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
    return lib


# every symbol the header declares (checked by tests/test_abi.py)
EXPORTS = ("bd_brute_overlaps", "bd_force","bd_force_prepare", "bd_force_slots", "bd_force_finish", "bd_maintain_tri", "bd_prepare_params", "bd_workspace_bytes", "bd_long_range_workspace_bytes",
           "bd_long_range_forces", "bd_short_range_forces", "bd_overlap_pass",
           "bd_max_sq_displacement", "bd_verlet_build", "bd_pairs_workspace_bytes", "bd_normals",
           "bd_step_tri", "bd_run_tri", "bd_step_verlet", "bd_run_verlet",
           "bd_tri_restore_delaunay", "bd_clear_status", "bd_tri_audit_geometry", "bd_build_info",
           "bd_integrate", "bd_tri_apply_crossings", "bd_tri_edge_inversion", "bd_tri_signed_area2",
           "bd_tri_delaunay_flags", "bd_tri_inverted_edge_flags", "bd_tri_flip_edges", "bd_tri_repair_inversions",
           "bd_tri_restore_delaunay_ex", "bd_overlap_correct", "bd_tri_copy", "bd_step_abp", "bd_run_abp",
           "bd_tri_build_workspace_bytes", "bd_tri_build_initial",
           "bd_long_range_workspace_bytes_for", "bd_force_sym_partial", "bd_force_sym_finish",
           "bd_integrate_noise", "bd_sym_shard", "bd_timing_enable", "bd_timing_read")
