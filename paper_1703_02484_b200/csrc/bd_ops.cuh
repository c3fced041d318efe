// bd_ops.cuh -- single-operation drivers: the reference's METHOD boundary.
//
// The step drivers (bd_drivers.cuh) fuse a whole step into one launch.  The
// reference also exposes the pieces of a step as public functions and
// methods, and its own tests drive them one at a time:
//
//   dynamics.integrate            dynamics.py:73-94
//   dynamics.correct_overlaps     dynamics.py:97-133
//   PeriodicTriangulation.apply_crossings        triangulation.py:166-177
//                        .signed_area2           :186-191
//                        .delaunay_flags         :226-229
//                        .inverted_edge_flags    :231-234
//                        .edge_inversion_present :240-250
//                        .flip_edge              :254-302
//                        .restore_delaunay       :319-334 (bd_step.cuh)
//                        .repair_inversions      :336-363
//
// Each op below runs the SAME phase functions the fused step uses
// (bd_step.cuh), so testing an op against the reference tests the step's
// building block.  Ops report through a small device int64 result array;
// the layout of each is documented at the op (and in include/bd_b200.h).
#pragma once

#include "bd_drivers.cuh"

namespace bd {

template <class X>
BD_HD void op_enter(X& x, Ctx& c) {
    if (x.leader()) {
        for (int k = 0; k < 8; ++k) c.w.ctl->red[k] = 0;
        c.w.ctl->status = 0;
        c.w.ctl->err_i = 0;
        c.w.ctl->err_k = 0;
        c.w.ctl->scratch[0] = ~0ull;  // first bad index of check_finite
        c.w.ctl->scratch[1] = ~0ull;
    }
    x.sync();
}

// integrate: res = {status, n_crossed, err_i}; crossings (n,2) int64 (may be
// null); noise (n,2) caller-drawn standard normals (null: the counter noise of
// call *s.call, which then advances; given: the call counter is left alone)
template <class X>
BD_HD void op_integrate(X& x, Ctx& c, double dt, int64_t* crossings, int64_t* res, const double* noise = nullptr) {
    Red<X> R(x);
    op_enter(x, c);
    bd_stats_t st;
    if (check_finite(x, R, c, &st)) {  // StepFailure before any state change (dynamics.py:84-86)
        if (x.leader()) {
            res[0] = BD_ERR_STEPFAIL;
            res[1] = 0;
            res[2] = st.err_i;
        }
        return;
    }
    const u64 nc = ph_integrate(x, R, c, dt, crossings, noise);
    if (x.leader()) {
        if (!noise) *c.s.call = c.call + 1;
        res[0] = 0;
        res[1] = (int64_t)nc;
        res[2] = 0;
    }
}

// apply_crossings with int64 crossings (n,2): the reference's int8 cast makes
// only crossings mod 256 visible, which is what cross8 holds
template <class X>
BD_HD void op_apply_crossings(X& x, Ctx& c, const int64_t* crossings) {
    Red<X> R(x);
    op_enter(x, c);
    u64* r = R.open();
    for (int64_t i = x.tid(); i < 2 * c.p.n; i += x.nth()) {
        c.w.cross8[i] = (int8_t)crossings[i];
        R.add((u64)(crossings[i] != 0));
    }
    if (R.close(r)) ph_apply_crossings(x, c);  // `if not np.any(crossings): return`
}

// edge_inversion_present(prev = c.s.prev, curr = c.s.pos): res[0] = 0/1
template <class X>
BD_HD void op_edge_inversion(X& x, Ctx& c, int64_t* res) {
    Red<X> R(x);
    op_enter(x, c);
    const bool v = ph_edge_inversion(x, R, c);
    if (x.leader()) res[0] = v;
}

// signed_area2 per triangle
template <class X>
BD_HD void op_signed_area2(X& x, Ctx& c, double* area) {
    const bd_tri_t& T = c.s.tri;
    for (int64_t t = x.tid(); t < T.nt; t += x.nth()) {
        V2 xy[3];
        tri_xy(T, c.s.pos, c.p.L, t, xy);
        const double e1x = xy[1].x - xy[0].x, e1y = xy[1].y - xy[0].y;
        const double e2x = xy[2].x - xy[0].x, e2y = xy[2].y - xy[0].y;
        area[t] = e1x * e2y - e1y * e2x;
    }
}

// delaunay_flags (tol = c.p.tol) or inverted_edge_flags per edge
template <class X>
BD_HD void op_edge_flags(X& x, Ctx& c, bool inverted, uint8_t* flags) {
    const bd_tri_t& T = c.s.tri;
    for (int64_t e = x.tid(); e < T.ne; e += x.nth()) {
        V2 q[4];
        edge_quad(T, c.s.pos, c.p.L, e, q);
        flags[e] = inverted ? (uint8_t)(point_in_tri(q[3], q[0], q[1], q[2]) | point_in_tri(q[2], q[0], q[1], q[3]))
                            : (uint8_t)incircle(q[0], q[1], q[2], q[3], c.p.tol);
    }
}

// flip_edge for each listed edge, in list order (one thread: consecutive
// flips may share triangles).  res = {status, index of the failing edge}
template <class X>
BD_HD void op_flip_edges(X& x, Ctx& c, const int64_t* edges, int64_t count, int64_t* res) {
    op_enter(x, c);
    if (x.leader()) {
        res[0] = 0;
        res[1] = -1;
        for (int64_t j = 0; j < count; ++j) {
            const int64_t e = edges[j];
            const int rc = (e < 0 || e >= c.s.tri.ne) ? BD_ERR_FLIP : flip_edge(c.s.tri, e);
            if (rc) {
                res[0] = rc;
                res[1] = j;
                break;
            }
        }
    }
    x.sync();
}

// repair_inversions(positions = c.s.pos, prev = c.s.prev if use_prev):
// res = {status, flips, passes, needs_rollback}
template <class X>
BD_HD void op_repair_inversions(X& x, Ctx& c, int64_t max_passes, bool use_prev, int64_t* res) {
    Red<X> R(x);
    op_enter(x, c);
    int64_t flips = 0, passes = 0;
    const int rr = repair_inversions(x, R, c, max_passes, &flips, use_prev, &passes);
    if (x.leader()) {
        res[0] = rr < 0 ? (int64_t)c.w.ctl->status : 0;
        res[1] = flips;
        res[2] = passes;
        res[3] = rr == 1;
    }
}

// restore_delaunay(positions = c.s.pos, tol = c.p.tol): res = {status, passes}
template <class X>
BD_HD void op_restore_delaunay(X& x, Ctx& c, int64_t max_passes, int64_t* res) {
    Red<X> R(x);
    op_enter(x, c);
    const int64_t p = restore_delaunay(x, R, c, max_passes);
    if (x.leader()) {
        res[0] = p < 0 ? (int64_t)c.w.ctl->status : 0;
        res[1] = p;
    }
}

// correct_overlaps over a fixed pair list; flags OR-ed into c.s.overlap_flags
// (flags_out |= flags, dynamics.py:118-119); with_tri: crossings of every
// sweep feed apply_crossings (dynamics.py:126-129).  res = {status, sweeps}
template <class X>
BD_HD void op_correct_overlaps(X& x, Ctx& c, int64_t n_pairs, bool with_tri, int64_t* res) {
    Red<X> R(x);
    op_enter(x, c);
    const ListPairs lp{c.s.pair_a, c.s.pair_b, n_pairs};
    build_incidence(x, c.p.n, lp, c.w.inc_off, c.w.inc_cur, c.w.inc);
    const int64_t it = correct_overlaps(x, R, c, lp, with_tri);
    if (x.leader()) {
        res[0] = it < 0 ? (int64_t)c.w.ctl->status : 0;
        res[1] = it;
    }
}

}  // namespace bd
