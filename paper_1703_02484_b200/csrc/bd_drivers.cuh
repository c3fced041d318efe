// bd_drivers.cuh -- whole-step drivers (uniform control flow over phases).
//
//   step_tri_after_force : LongRangeSimulation.step (dynamics.py:191-274)
//                          after the all-pairs force kernel, with the composite
//                          force models: short-range Verlet force
//                          alone or added to the long-range force, the
//                          triangulation being the overlap neighbour provider;
//   step_verlet          : ShortRangeSimulation.step (dynamics.py:326-346).
#pragma once

#include "bd_verlet.cuh"

namespace bd {

// first receiver with a non-zero err sentinel -> SingularityError (forces.py:54-58)
template <class X>
BD_HD bool check_singular(X& x, Red<X>& R, Ctx& c, const int64_t* err, bd_stats_t* out) {
    u64* r = R.open();  // scratch[1] = ~0 since driver_enter / op_enter (only an error, which ends the step, lowers it)
    for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) {
        const bool bad = err[i] != 0;
        if (bad) x.umin(&c.w.ctl->scratch[1], (u64)i);
        R.add((u64)bad);
    }
    if (!R.close(r)) return false;
    if (x.leader()) {
        const int64_t i = (int64_t)c.w.ctl->scratch[1];
        c.w.ctl->status = BD_ERR_SINGULAR;
        c.w.ctl->err_i = (u64)i;
        c.w.ctl->err_k = (u64)(err[i] - 1);
        out->status = BD_ERR_SINGULAR;
        out->err_i = i;
        out->err_k = err[i] - 1;
    }
    x.sync();
    return true;
}

// non-finite force -> StepFailure (integrate, dynamics.py:84-86)
template <class X>
BD_HD bool check_finite(X& x, Red<X>& R, Ctx& c, bd_stats_t* out) {
    u64* r = R.open();  // scratch[0] = ~0 since driver_enter / op_enter
    for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) {
        const bool bad = !(isfinite(c.s.force[2 * i]) && isfinite(c.s.force[2 * i + 1]));
        if (bad) x.umin(&c.w.ctl->scratch[0], (u64)i);
        R.add((u64)bad);
    }
    if (!R.close(r)) return false;
    if (x.leader()) {
        c.w.ctl->status = BD_ERR_STEPFAIL;
        c.w.ctl->err_i = c.w.ctl->scratch[0];
        out->status = BD_ERR_STEPFAIL;
        out->err_i = (int64_t)c.w.ctl->scratch[0];
    }
    x.sync();
    return true;
}

// check_singular (when err is given) + check_finite + save_state
// (triangulation.py:158-160, with the image counters; `backup`) as ONE phase: the
// checks only read, the backup only writes the backup arrays, so a single
// barrier serves all three (the singular check keeps precedence)
template <class X>
BD_HD bool check_and_backup(X& x, Red<X>& R, Ctx& c, const int64_t* err, bd_stats_t* out, bool backup = true) {
    u64* r = R.open();  // scratch[0] / scratch[1] = ~0 since driver_enter
    for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) {
        const bool bs = err && err[i] != 0;
        const bool bf = !(isfinite(c.s.force[2 * i]) && isfinite(c.s.force[2 * i + 1]));
        if (bs) x.umin(&c.w.ctl->scratch[1], (u64)i);
        if (bf) x.umin(&c.w.ctl->scratch[0], (u64)i);
        R.add((u64)bs | ((u64)bf << 32));
    }
    if (backup) {
        ph_tri_copy(x, c.s.tri, c.s.tri_backup);
        if (c.s.image)
            for (int64_t i = x.tid(); i < 2 * c.p.n; i += x.nth()) c.w.image_bk[i] = c.s.image[i];
    }
    const u64 v = R.close(r);
    if (v & 0xffffffffull) {
        if (x.leader()) {
            const int64_t i = (int64_t)c.w.ctl->scratch[1];
            c.w.ctl->status = BD_ERR_SINGULAR;
            c.w.ctl->err_i = (u64)i;
            c.w.ctl->err_k = (u64)(err[i] - 1);
            out->status = BD_ERR_SINGULAR;
            out->err_i = i;
            out->err_k = err[i] - 1;
        }
        x.sync();
        return true;
    }
    if (v >> 32) {
        if (x.leader()) {
            c.w.ctl->status = BD_ERR_STEPFAIL;
            c.w.ctl->err_i = c.w.ctl->scratch[0];
            out->status = BD_ERR_STEPFAIL;
            out->err_i = (int64_t)c.w.ctl->scratch[0];
        }
        x.sync();
        return true;
    }
    return false;
}

template <class X>
BD_HD bool driver_enter(X& x, Red<X>& R, Ctx& c, bd_stats_t* out) {
    if (x.leader()) {
        for (int k = 0; k < 8; ++k) c.w.ctl->red[k] = 0;
        c.w.ctl->scratch[0] = ~0ull;  // first bad index of check_finite / check_singular
        c.w.ctl->scratch[1] = ~0ull;
    }
    x.sync();
    if (x.ld(&c.w.ctl->status)) {  // an earlier step failed: this one does not run
        if (x.leader()) out->status = -1;
        return false;
    }
    return true;
}

// LongRangeSimulation.step after the all-pairs force (dynamics.py:196-274).
// s.force holds F_LR (force_mode LR / LRSR) from the all-pairs kernel.
// phase timers for the breakdown in bd_stats_t.work (leader's clock, between barriers)
template <class X>
BD_HD int maintain_t(X& x, Red<X>& R, Ctx& c, int64_t* repairs, int64_t* flip_passes) {
    const int64_t t0 = now_ns();
    const int m = maintain(x, R, c, repairs, flip_passes);
    c.work[WK_T_MAINTAIN] += now_ns() - t0;
    return m;
}

template <class X, class PS>
BD_HD int64_t correct_overlaps_t(X& x, Red<X>& R, Ctx& c, const PS& ps, bool tri, bool edge_inc = false) {
    const int64_t t0 = now_ns(), ti0 = c.work[WK_T_INCIDENCE];
    const int64_t r = correct_overlaps(x, R, c, ps, tri, edge_inc);
    c.work[WK_T_OVERLAP] += now_ns() - t0 - (c.work[WK_T_INCIDENCE] - ti0);  // lazy incidence builds: their own timer
    return r;
}

template <class X>
BD_HD void step_tri_after_force(X& x, Ctx& c, bd_stats_t* out) {
    Red<X> R(x);
    const int64_t t_enter = now_ns();
    if (!driver_enter(x, R, c, out)) return;
    const int64_t rebuilds0 = c.s.vl_meta ? c.s.vl_meta[2] : 0;
    if (c.p.force_mode == BD_FORCE_LRSR && check_singular(x, R, c, c.s.force_err, out)) return;
    if (c.p.force_mode != BD_FORCE_LR) {
        // short-range force over a Verlet list kept fresh by the rebuild rule
        const bool stale = vl_stale(x, R, c);
        if (stale && !vl_rebuild(x, R, c, 0.0)) {
            if (x.leader()) out->status = BD_ERR_CAPACITY;
            return;
        }
        sr_forces(x, c, c.w.sr_force, c.w.sr_err);
        if (check_singular(x, R, c, c.w.sr_err, out)) return;
        const bool add = c.p.force_mode == BD_FORCE_LRSR;
        for (int64_t i = x.tid(); i < 2 * c.p.n; i += x.nth())
            c.s.force[i] = add ? c.s.force[i] + c.w.sr_force[i] : c.w.sr_force[i];
        x.sync();
    }
    // LR: the long-range singularity check here; + check_finite + save_state
    if (check_and_backup(x, R, c, c.p.force_mode == BD_FORCE_LR ? c.s.force_err : nullptr, out)) return;

    double dt_try = c.p.dt;
    int64_t rollbacks = 0, iters = 0, repairs = 0, flip_passes = 0;
    bool failed = false;
    c.work[WK_T_PRE] = now_ns() - t_enter;
    for (;;) {
        const int64_t t_int = now_ns();
        const u64 nc = ph_integrate(x, R, c, dt_try);
        c.call++;
        if (nc) ph_apply_crossings(x, c);
        c.work[WK_T_INTEGRATE] += now_ns() - t_int;
        repairs = 0;
        flip_passes = 0;
        int m = maintain_t(x, R, c, &repairs, &flip_passes);
        if (m < 0) break;
        failed = m == 1;
        if (!failed) {
            iters = 0;
            for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) c.s.overlap_flags[i] = 0;
            int64_t outer;
            for (outer = 0; outer < c.p.max_overlap_iters; ++outer) {
                const int64_t ri = correct_overlaps_t(x, R, c, EdgePairs{c.s.tri.edge_v, c.s.tri.ne}, true, true);
                if (ri < 0) break;
                iters += ri;
                if (ri == 0) break;
                m = maintain_t(x, R, c, &repairs, &flip_passes);
                if (m < 0) break;
                failed = m == 1;
                if (failed) break;
            }
            if (x.ld(&c.w.ctl->status)) break;
            if (outer == c.p.max_overlap_iters) {
                set_error(x, c, BD_ERR_NONCONV, 0, 0);
                x.sync();
                break;
            }
        }
        if (!failed) break;
        rollbacks++;
        if (rollbacks > c.p.max_rollbacks) {
            set_error(x, c, BD_ERR_STEPFAIL, rollbacks, 0);
            x.sync();
            break;
        }
        // restore_prev + restore_state, dt halving (dynamics.py:259-261)
        for (int64_t i = x.tid(); i < 2 * c.p.n; i += x.nth()) c.s.pos[i] = c.s.prev[i];
        if (c.s.image)
            for (int64_t i = x.tid(); i < 2 * c.p.n; i += x.nth()) c.s.image[i] = c.w.image_bk[i];
        ph_tri_copy(x, c.s.tri_backup, c.s.tri);
        c.inc_flips = -1;  // edge_v restored: the incidence lists are stale
        x.sync();
        dt_try *= 0.5;
    }
    // n_overlapping
    u64* r = R.open();
    for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) R.add((u64)c.s.overlap_flags[i]);
    const u64 nov = R.close(r);
    if (x.leader()) {
        out->rebuilds = c.s.vl_meta ? c.s.vl_meta[2] - rebuilds0 : 0;
        out->dt_used = dt_try;
        out->overlap_iterations = iters;
        out->flip_passes = flip_passes;
        out->inversion_repairs = repairs;
        out->rollbacks = rollbacks;
        out->n_overlapping = (int64_t)nov;
        out->status = (int64_t)c.w.ctl->status;
        out->err_i = (int64_t)c.w.ctl->err_i;
        out->err_k = (int64_t)c.w.ctl->err_k;
        out->calls = (int64_t)c.call;
        c.work[WK_T_TOTAL] = now_ns() - t_enter;
        for (int k = 0; k < WK_N; ++k) out->work[k] = c.work[k];
        *c.s.call = c.call;
    }
}


// _VerletNeighborMixin._overlap_rounds (dynamics.py:290-304): correct over
// the overlap candidates; rebuild (candidates within `margin`) and repeat
// while the motion since the snapshot exceeds skin/2.  Returns the sweeps.
template <class X>
BD_HD int64_t overlap_rounds(X& x, Red<X>& R, Ctx& c, double margin) {
    int64_t iters = 0, round;
    for (round = 0; round < c.p.max_overlap_iters; ++round) {
        const SubsetPairs sp{c.s.pair_a, c.s.pair_b, c.w.ov_idx, (int64_t)x.ld((const u64*)&c.s.vl_meta[3])};
        const int64_t t0 = now_ns();
        build_incidence(x, c.p.n, sp, c.w.inc_off, c.w.inc_cur, c.w.inc, c.work);
        c.work[WK_T_INCIDENCE] += now_ns() - t0;
        const int64_t ri = correct_overlaps_t(x, R, c, sp, false);
        if (ri < 0) break;
        iters += ri;
        if (!vl_stale(x, R, c)) break;
        if (!vl_rebuild(x, R, c, margin)) break;
    }
    if (!x.ld(&c.w.ctl->status) && round == c.p.max_overlap_iters) {
        set_error(x, c, BD_ERR_NONCONV, 0, 0);
        x.sync();
    }
    return iters;
}

template <class X>
BD_HD void verlet_stats(X& x, Red<X>& R, Ctx& c, bd_stats_t* out, int64_t rebuilds0, int64_t iters,
                        int64_t t_enter) {
    u64* r = R.open();
    for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) R.add((u64)c.s.overlap_flags[i]);
    const u64 nov = R.close(r);
    if (x.leader()) {
        out->rebuilds = c.s.vl_meta[2] - rebuilds0;
        out->dt_used = c.p.dt;
        out->overlap_iterations = iters;
        out->flip_passes = 0;
        out->inversion_repairs = 0;
        out->rollbacks = 0;
        out->n_overlapping = (int64_t)nov;
        out->status = (int64_t)c.w.ctl->status;
        out->err_i = (int64_t)c.w.ctl->err_i;
        out->err_k = (int64_t)c.w.ctl->err_k;
        out->calls = (int64_t)c.call;
        c.work[WK_T_TOTAL] = now_ns() - t_enter;
        for (int k = 0; k < WK_N; ++k) out->work[k] = c.work[k];
        *c.s.call = c.call;
    }
}

// ShortRangeSimulation.step (dynamics.py:326-346): fresh list, short-range
// force, integrate, overlap rounds over the overlap candidates with list
// rebuilds whenever motion since the snapshot exceeds skin/2.
template <class X>
BD_HD void step_verlet(X& x, Ctx& c, bd_stats_t* out) {
    Red<X> R(x);
    const int64_t t_enter = now_ns();
    if (!driver_enter(x, R, c, out)) return;
    const int64_t rebuilds0 = c.s.vl_meta[2];
    const double margin = c.p.sigma + c.p.skin;
    if (vl_stale(x, R, c) && !vl_rebuild(x, R, c, margin)) {
        if (x.leader()) out->status = BD_ERR_CAPACITY;
        return;
    }
    sr_forces(x, c, c.s.force, c.s.force_err);
    if (check_and_backup(x, R, c, c.s.force_err, out, false)) return;  // check_singular + check_finite
    ph_integrate(x, R, c, c.p.dt);
    c.call++;
    for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) c.s.overlap_flags[i] = 0;
    const int64_t iters = overlap_rounds(x, R, c, margin);
    verlet_stats(x, R, c, out, rebuilds0, iters, t_enter);
}

// AbpSimulation.step move (dynamics.py:378-390): prev <- pos; pos =
// wrap(pos + (V0 dt) (cos theta, sin theta)); theta += sqrt(2 D_r dt) xi with
// xi element i of one normals(n) call (pair i/2, component i%2), clamped
// when clamp_angle_noise.  Crossings feed the image counters (MSD).
template <class X>
BD_HD void ph_abp_move(X& x, Ctx& c) {
    const double L = c.p.L, s = c.p.abp_speed * c.p.dt;
    const double ang_scale = sqrt(2.0 * c.p.abp_rot_diffusion * c.p.dt);
    double* pos = c.s.pos;
    for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) {
        const double th = c.s.angles[i];
        double h[2];
#if defined(__CUDA_ARCH__)
        sincos(th, &h[1], &h[0]);
#else
        h[0] = cos(th);
        h[1] = sin(th);
#endif
        for (int k = 0; k < 2; ++k) {
            const double p0 = pos[2 * i + k];
            c.s.prev[2 * i + k] = p0;
            const double nw = p0 + s * h[k];
            const double w = wrap1(nw, L);
            pos[2 * i + k] = w;
            if (c.s.image) c.s.image[2 * i + k] += (int32_t)rint((nw - w) / L);
        }
        double z0, z1;
        normal_pair(c.p.seed, c.p.stream, c.call, (uint64_t)(i >> 1), 0, z0, z1);
        double z = (i & 1) ? z1 : z0;
        if (c.p.abp_clamp_angle) z = clampd(z, c.p.clamp);
        c.s.angles[i] = th + ang_scale * z;
    }
    x.sync();
}

// AbpSimulation.step (dynamics.py:368-399): fresh list, ballistic move +
// angle diffusion, overlap rounds with candidates within sigma + skin.
template <class X>
BD_HD void step_abp(X& x, Ctx& c, bd_stats_t* out) {
    Red<X> R(x);
    const int64_t t_enter = now_ns();
    if (!driver_enter(x, R, c, out)) return;
    const int64_t rebuilds0 = c.s.vl_meta[2];
    const double margin = c.p.r_list;  // overlap_margin = r_list = sigma + skin (dynamics.py:366-367)
    if (vl_stale(x, R, c) && !vl_rebuild(x, R, c, margin)) {
        if (x.leader()) out->status = BD_ERR_CAPACITY;
        return;
    }
    ph_abp_move(x, c);
    c.call++;
    for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) c.s.overlap_flags[i] = 0;
    const int64_t iters = overlap_rounds(x, R, c, margin);
    verlet_stats(x, R, c, out, rebuilds0, iters, t_enter);
}

}  // namespace bd
