// bd_step.cuh -- device-resident step driver (one source, three policies).
//
// Restates LongRangeSimulation.step (dynamics.py:191-274) and its callees
// (integrate dynamics.py:73-94, correct_overlaps :97-133, the triangulation
// maintenance triangulation.py:166-363) as uniform phases over particles,
// edges and triangles, separated by barriers (see bd_exec.cuh).
//
// Bit-exactness: every floating-point expression follows the reference's
// evaluation order; per-particle sums that the reference accumulates in
// ascending pair order are gathered per particle over an incidence list
// sorted by pair index, so the GPU result is bit-identical to the reference
// (and to oracle/bd_oracle.c) on the same inputs and noise.
#pragma once

#include "bd_allpairs_sym.cuh"
#include "bd_exec.cuh"

namespace bd {

enum : uint8_t { ES_NONE = 0, ES_UND = 1, ES_SEL = 2, ES_REM = 3 };

// workspace carve-up (device pointers)
struct Ws {
    Ctl* ctl;
    double* contrib;   // (items,2) per-pair bounce displacement of the current sweep
    uint8_t* estat;    // (ne) flag / selection status
    uint8_t* eovl;     // (items) pair overlapping this sweep
    uint8_t* tinv;     // (nt) triangle inverted
    int8_t* cross8;    // (n,2) crossings mod 256 (all apply_crossings needs)
    int32_t* image_bk; // (n,2)
    int32_t* inc_off;  // (n+1) CSR offsets of the overlap neighbour pairs per vertex
    int32_t* inc_cur;  // (n) fill cursors
    int32_t* inc;      // (2 items) incident pairs, ascending per vertex
    int32_t* wl0;      // (ne) restore_delaunay worklist: flagged edges
    int32_t* wl1;      // (ne) restore_delaunay worklist: edges to re-evaluate
    uint32_t* stamp;   // (ne) worklist dedup stamps
    uint32_t* ewin;    // (ne) LFMIS: round stamp of the selection of each edge (ph_select_and_flip)
    uint32_t* vhit;    // (n) correct_overlaps: sweep stamp of the particles with an overlapping pair
    double* src4;      // all-pairs scratch (packed sources / sorted FAST workspace)
    // Verlet list (forces.py:67-156)
    int32_t* cell_id;    // (n)
    int32_t* cell_start; // (ncells+1)
    int32_t* cell_cur;   // (ncells)
    int32_t* corder;     // (n) stable cell order
    int32_t* pcnt;       // (max(5 n, ncells)+1) pairs per (cell, segment, particle) item (or per row) -> offsets
    int32_t* vinc_off;   // (n+1) CSR of Verlet pairs per particle
    int32_t* vinc_cur;   // (n)
    int32_t* vinc;       // (2 P)
    int32_t* ov_idx;     // (P) overlap-candidate subset (ShortRangeSimulation)
    int64_t* sr_err;     // (n)
    double* sr_force;    // (n,2) short-range contribution
};

BD_HD int64_t align_up(int64_t x) { return (x + 255) & ~(int64_t)255; }

BD_HD int64_t ncells_of(const bd_params_t& p) { return p.ncx > 0 ? p.ncx * p.ncx : 0; }

// layout of bd_workspace_bytes(); offsets relative to the workspace base
struct WsLayout {
    int64_t ctl, contrib, estat, eovl, tinv, cross8, image_bk, inc_off, inc_cur, inc, wl0, wl1, stamp, ewin, vhit, src4;
    int64_t cell_id, cell_start, cell_cur, corder, pcnt, vinc_off, vinc_cur, vinc, ov_idx, sr_err, sr_force, total;
};

BD_HD WsLayout ws_layout(const bd_params_t& p, int64_t ne, int64_t nt) {
    const int64_t n = p.n, P = p.pair_capacity > 0 ? p.pair_capacity : 0, nc = ncells_of(p);
    const int64_t items = ne > P ? ne : P;
    WsLayout l;
    int64_t o = 0;
    l.ctl = o; o = align_up(o + (int64_t)sizeof(Ctl));
    l.contrib = o; o = align_up(o + 16 * items);
    l.estat = o; o = align_up(o + ne);
    l.eovl = o; o = align_up(o + items);
    l.tinv = o; o = align_up(o + nt);
    l.cross8 = o; o = align_up(o + 2 * n);
    l.image_bk = o; o = align_up(o + 8 * n);
    l.inc_off = o; o = align_up(o + 4 * (n + 1));
    l.inc_cur = o; o = align_up(o + 4 * n);
    l.inc = o; o = align_up(o + 8 * items);
    l.wl0 = o; o = align_up(o + 4 * ne);
    l.wl1 = o; o = align_up(o + 4 * ne);
    l.stamp = o; o = align_up(o + 4 * ne);
    l.ewin = o; o = align_up(o + 4 * ne);
    l.vhit = o; o = align_up(o + 4 * n);
    // all-pairs scratch: packed double4 sources (EXACT) or the sorted FAST workspace
    {
        int64_t f = fast_ws_bytes(n) > 32 * n ? fast_ws_bytes(n) : 32 * n;
        if (p.lr_precision == BD_LR_FAST_SYM) f = sym_ws_bytes(n);
        l.src4 = o; o = align_up(o + f);
    }
    l.cell_id = o; o = align_up(o + (P ? 4 * n : 0));
    l.cell_start = o; o = align_up(o + (P ? 4 * (nc + 1) : 0));
    l.cell_cur = o; o = align_up(o + (P ? 4 * nc : 0));
    l.corder = o; o = align_up(o + (P ? 4 * n : 0));
    l.pcnt = o; o = align_up(o + (P ? 4 * ((nc > 5 * n ? nc : 5 * n) + 1) : 0));
    l.vinc_off = o; o = align_up(o + (P ? 4 * (n + 1) : 0));
    l.vinc_cur = o; o = align_up(o + (P ? 4 * n : 0));
    l.vinc = o; o = align_up(o + 8 * P);
    l.ov_idx = o; o = align_up(o + 4 * P);
    l.sr_err = o; o = align_up(o + (P ? 8 * n : 0));
    l.sr_force = o; o = align_up(o + (P ? 16 * n : 0));
    l.total = o;
    return l;
}

BD_HD Ws ws_carve(void* base, const bd_params_t& p, int64_t ne, int64_t nt) {
    WsLayout l = ws_layout(p, ne, nt);
    char* b = (char*)base;
    Ws w;
    w.ctl = (Ctl*)(b + l.ctl);
    w.contrib = (double*)(b + l.contrib);
    w.estat = (uint8_t*)(b + l.estat);
    w.eovl = (uint8_t*)(b + l.eovl);
    w.tinv = (uint8_t*)(b + l.tinv);
    w.cross8 = (int8_t*)(b + l.cross8);
    w.image_bk = (int32_t*)(b + l.image_bk);
    w.inc_off = (int32_t*)(b + l.inc_off);
    w.inc_cur = (int32_t*)(b + l.inc_cur);
    w.inc = (int32_t*)(b + l.inc);
    w.wl0 = (int32_t*)(b + l.wl0);
    w.wl1 = (int32_t*)(b + l.wl1);
    w.stamp = (uint32_t*)(b + l.stamp);
    w.ewin = (uint32_t*)(b + l.ewin);
    w.vhit = (uint32_t*)(b + l.vhit);
    w.src4 = (double*)(b + l.src4);
    w.cell_id = (int32_t*)(b + l.cell_id);
    w.cell_start = (int32_t*)(b + l.cell_start);
    w.cell_cur = (int32_t*)(b + l.cell_cur);
    w.corder = (int32_t*)(b + l.corder);
    w.pcnt = (int32_t*)(b + l.pcnt);
    w.vinc_off = (int32_t*)(b + l.vinc_off);
    w.vinc_cur = (int32_t*)(b + l.vinc_cur);
    w.vinc = (int32_t*)(b + l.vinc);
    w.ov_idx = (int32_t*)(b + l.ov_idx);
    w.sr_err = (int64_t*)(b + l.sr_err);
    w.sr_force = (double*)(b + l.sr_force);
    return w;
}

// Work counters of one step (uniform across threads: every thread runs the
// same phase sequence), reported in bd_stats_t.work[] so the host can turn
// them into algorithmic bytes (bench.py "maintain_roofline").
enum {
    WK_INTEGRATE = 0,  // integrate passes (attempts)
    WK_APPLY_CROSS,    // apply_crossings passes
    WK_EDGE_INV,       // edge-inversion (pass-through) checks
    WK_FLAG_PASS,      // per-edge predicate passes (in-circle / inversion flags)
    WK_AREA_PASS,      // per-triangle signed-area passes
    WK_LFMIS_ROUND,    // independent-set selection rounds
    WK_FLIPS,          // edges flipped
    WK_OVL_PASS,       // overlap passes over the pair list (incl. the final clean one)
    WK_OVL_APPLY,      // overlap gather/apply passes
    WK_INCIDENCE,      // incidence-list builds
    WK_VL_REBUILD,     // Verlet list rebuilds
    WK_SR_FORCE,       // short-range force evaluations
    WK_T_MAINTAIN,     // ns in pass-through check + inversion repair + Delaunay restoration
    WK_T_OVERLAP,      // ns in overlap sweeps
    WK_T_INCIDENCE,    // ns in incidence-list builds
    WK_T_TOTAL,        // ns from driver entry to exit
    WK_T_VERLET,       // ns in Verlet list rebuilds (cell sort + ordered pair fill)
    WK_T_SR_FORCE,     // ns in short-range force evaluations
    WK_T_PRE,          // ns before the first integrate (force checks, SR force, rollback backup)
    WK_T_INTEGRATE,    // ns in integrate + its apply_crossings
    WK_FLAG_EDGES_WL,  // edges re-evaluated by worklist passes of restore_delaunay
    WK_N
};

static_assert(WK_N <= 24, "bd_stats_t.work has 24 words");

struct Ctx {
    bd_params_t p;
    bd_state_t s;
    Ws w;
    uint64_t call;
    int64_t work[WK_N];
    int64_t inc_flips;  // work[WK_FLIPS] when the edge incidence lists were last built (-1: stale)
};

BD_HD void ctx_init_work(Ctx& c) {
    for (int k = 0; k < WK_N; ++k) c.work[k] = 0;
    c.inc_flips = -1;
}

// device wall clock (ns) for the phase breakdown; 0 on the host emulation
BD_HD int64_t now_ns() {
#if defined(__CUDA_ARCH__)
    // only the leader's timers are reported (bd_stats_t.work); the other
    // threads skip the (slow) global-timer read
    if (threadIdx.x != 0 || blockIdx.x != 0) return 0;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (int64_t)t;
#else
    return 0;
#endif
}

template <class X>
BD_HD void set_error(X& x, Ctx& c, u64 code, int64_t i, int64_t k) {
    if (x.cas(&c.w.ctl->status, 0, code) == 0) {
        c.w.ctl->err_i = (u64)i;
        c.w.ctl->err_k = (u64)k;
    }
}

// ---------------------------------------------------------------------------
// small per-element helpers

BD_HD double tri_coord(const bd_tri_t& T, const double* pos, double L, int64_t t, int k, int c) {
    return pos[2 * (int64_t)T.tri_v[3 * t + k] + c] + (double)T.tri_shift[6 * t + 2 * k + c] * L;
}

BD_HD void tri_xy(const bd_tri_t& T, const double* pos, double L, int64_t t, V2 xy[3]) {
    for (int k = 0; k < 3; ++k) {
        xy[k].x = tri_coord(T, pos, L, t, k, 0);
        xy[k].y = tri_coord(T, pos, L, t, k, 1);
    }
}

// edge_quads, triangulation.py:193-222
BD_HD void edge_quad(const bd_tri_t& T, const double* pos, double L, int64_t e, V2 q[4]) {
    const int64_t tl = T.edge_tri[2 * e], tr = T.edge_tri[2 * e + 1];
    const int ol = T.edge_opp[2 * e], orr = T.edge_opp[2 * e + 1];
    const int a_sl = (ol + 1) % 3, b_sl = (ol + 2) % 3, a_sr = (orr + 2) % 3;
    const int8_t* sl = T.tri_shift + 6 * tl;
    const int8_t* sr = T.tri_shift + 6 * tr;
    q[0] = emb(pos, T.tri_v[3 * tl + a_sl], (double)sl[2 * a_sl], (double)sl[2 * a_sl + 1], L);
    q[1] = emb(pos, T.tri_v[3 * tl + b_sl], (double)sl[2 * b_sl], (double)sl[2 * b_sl + 1], L);
    q[2] = emb(pos, T.tri_v[3 * tl + ol], (double)sl[2 * ol], (double)sl[2 * ol + 1], L);
    const double dlx = (double)sl[2 * a_sl] - (double)sr[2 * a_sr];
    const double dly = (double)sl[2 * a_sl + 1] - (double)sr[2 * a_sr + 1];
    q[3] = emb(pos, T.tri_v[3 * tr + orr], (double)sr[2 * orr] + dlx, (double)sr[2 * orr + 1] + dly, L);
}

// one side of _crossed_edges (triangulation.py:365-382): did the path of the
// vertex in slot k of triangle t cross the opposite edge?
BD_HD bool crossed_side(const bd_tri_t& T, const double* pos, const double* prv, const bd_params_t& p,
                        int64_t t, int k) {
    V2 xy[3];
    tri_xy(T, pos, p.L, t, xy);
    const int64_t w = T.tri_v[3 * t + k];
    const double sx = mi_exact(pos[2 * w] - prv[2 * w], p), sy = mi_exact(pos[2 * w + 1] - prv[2 * w + 1], p);
    V2 ps;
    ps.x = xy[k].x - sx;
    ps.y = xy[k].y - sy;
    return seg_intersect(ps, xy[k], xy[(k + 1) % 3], xy[(k + 2) % 3]);
}

// flip_edge + _relink, triangulation.py:254-302 (conflict-free flips may run concurrently)
// An outer edge of one selected quad can be an outer edge of another one
// flipped concurrently: each flip rewrites only the side that referenced
// its own old triangle, but finding that side reads the other side's word,
// which the other flip may be writing.  The side is therefore claimed with
// a compare-and-swap on side 0 (the other flip's triangles never equal
// ours, so the outcome does not depend on the interleaving, and no plain
// read races a plain write: compute-sanitizer racecheck clean).
BD_HD void relink(bd_tri_t& T, int64_t edge, int32_t old_tri, int32_t new_tri, int8_t opp) {
#if defined(__CUDA_ARCH__)
    const int side = atomicCAS(&T.edge_tri[2 * edge], old_tri, new_tri) == old_tri ? 0 : 1;
    if (side) T.edge_tri[2 * edge + 1] = new_tri;
#else
    const int side = T.edge_tri[2 * edge] == old_tri ? 0 : 1;
    T.edge_tri[2 * edge + side] = new_tri;
#endif
    T.edge_opp[2 * edge + side] = opp;
}

BD_HD int flip_edge(bd_tri_t& T, int64_t e) {
    const int32_t tl = T.edge_tri[2 * e], tr = T.edge_tri[2 * e + 1];
    if (tl == tr) return BD_ERR_FLIP;
    const int ol = T.edge_opp[2 * e], orr = T.edge_opp[2 * e + 1];
    const int a_sl = (ol + 1) % 3, b_sl = (ol + 2) % 3, b_sr = (orr + 1) % 3, a_sr = (orr + 2) % 3;
    const int32_t va = T.tri_v[3 * tl + a_sl], vb = T.tri_v[3 * tl + b_sl];
    const int32_t vc = T.tri_v[3 * tl + ol], vd = T.tri_v[3 * tr + orr];
    int32_t sa[2], sb[2], sc[2], sd[2];
    for (int c = 0; c < 2; ++c) {
        sa[c] = T.tri_shift[6 * tl + 2 * a_sl + c];
        sb[c] = T.tri_shift[6 * tl + 2 * b_sl + c];
        sc[c] = T.tri_shift[6 * tl + 2 * ol + c];
        sd[c] = (int32_t)T.tri_shift[6 * tr + 2 * orr + c] + (sa[c] - (int32_t)T.tri_shift[6 * tr + 2 * a_sr + c]);
    }
    const int32_t e_bc = T.tri_edge[3 * tl + a_sl], e_ca = T.tri_edge[3 * tl + b_sl];
    const int32_t e_ad = T.tri_edge[3 * tr + b_sr], e_db = T.tri_edge[3 * tr + a_sr];
    const int64_t ids[5] = {e, e_bc, e_ca, e_ad, e_db};
    for (int i = 0; i < 5; ++i)
        for (int j = i + 1; j < 5; ++j)
            if (ids[i] == ids[j]) return BD_ERR_FLIP;
    T.tri_v[3 * tl] = vc; T.tri_v[3 * tl + 1] = va; T.tri_v[3 * tl + 2] = vd;
    T.tri_v[3 * tr] = vd; T.tri_v[3 * tr + 1] = vb; T.tri_v[3 * tr + 2] = vc;
    for (int c = 0; c < 2; ++c) {
        T.tri_shift[6 * tl + c] = 0;
        T.tri_shift[6 * tl + 2 + c] = (int8_t)(sa[c] - sc[c]);
        T.tri_shift[6 * tl + 4 + c] = (int8_t)(sd[c] - sc[c]);
        T.tri_shift[6 * tr + c] = 0;
        T.tri_shift[6 * tr + 2 + c] = (int8_t)(sb[c] - sd[c]);
        T.tri_shift[6 * tr + 4 + c] = (int8_t)(sc[c] - sd[c]);
    }
    T.tri_edge[3 * tl] = e_ad; T.tri_edge[3 * tl + 1] = (int32_t)e; T.tri_edge[3 * tl + 2] = e_ca;
    T.tri_edge[3 * tr] = e_bc; T.tri_edge[3 * tr + 1] = (int32_t)e; T.tri_edge[3 * tr + 2] = e_db;
    T.edge_v[2 * e] = vc; T.edge_v[2 * e + 1] = vd;
    T.edge_tri[2 * e] = tr; T.edge_tri[2 * e + 1] = tl;
    T.edge_opp[2 * e] = 1; T.edge_opp[2 * e + 1] = 1;
    relink(T, e_ca, tl, tl, 2);
    relink(T, e_ad, tr, tl, 0);
    relink(T, e_bc, tl, tr, 0);
    relink(T, e_db, tr, tr, 2);
    return BD_OK;
}

// ---------------------------------------------------------------------------
// phases

// dst[0, bytes) = src[0, bytes) by the policy's threads (no barrier)
template <class X>
BD_HD void copy_bytes(X& x, void* dst, const void* src, int64_t bytes) {
    unsigned char* d = (unsigned char*)dst;
    const unsigned char* s = (const unsigned char*)src;
    int64_t body = 0;
    if ((((uintptr_t)d | (uintptr_t)s) & 15) == 0) {
        body = bytes & ~(int64_t)15;
        struct alignas(16) V16 {
            unsigned long long a, b;
        };
        for (int64_t i = x.tid(); i < body / 16; i += x.nth()) ((V16*)d)[i] = ((const V16*)s)[i];
    }
    for (int64_t i = body + x.tid(); i < bytes; i += x.nth()) d[i] = s[i];
}

// copy the six triangulation arrays a -> b (save_state / restore_state)
template <class X>
BD_HD void ph_tri_copy(X& x, const bd_tri_t& a, bd_tri_t& b) {
    // each array as a flat byte range, 16 bytes per thread and step where
    // both ends are 16-byte aligned (the device and shared-memory arrays are)
    copy_bytes(x, b.tri_v, a.tri_v, 12 * a.nt);
    copy_bytes(x, b.tri_edge, a.tri_edge, 12 * a.nt);
    copy_bytes(x, b.tri_shift, a.tri_shift, 6 * a.nt);
    copy_bytes(x, b.edge_v, a.edge_v, 8 * a.ne);
    copy_bytes(x, b.edge_tri, a.edge_tri, 8 * a.ne);
    copy_bytes(x, b.edge_opp, a.edge_opp, 2 * a.ne);
}

// integrate (dynamics.py:73-94) fused with the crossing bookkeeping; returns #particles that crossed
template <class X>
BD_HD u64 ph_integrate(X& x, Red<X>& R, Ctx& c, double dt, int64_t* cross64 = nullptr,
                       const double* noise = nullptr) {
    c.work[WK_INTEGRATE]++;
    u64* r = R.open();
    const double L = c.p.L, scale = sqrt(c.p.diffusion * dt), clamp = c.p.clamp;
    double* pos = c.s.pos;
    for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) {
        double z0, z1;
        if (noise) {  // caller-drawn normals (the reference's own rng.normals((n, 2)))
            z0 = noise[2 * i];
            z1 = noise[2 * i + 1];
        } else {
            normal_pair(c.p.seed, c.p.stream, c.call, (uint64_t)i, 0, z0, z1);
        }
        const double z[2] = {clampd(z0, clamp), clampd(z1, clamp)};
        int crossed = 0;
        for (int k = 0; k < 2; ++k) {
            const double p0 = pos[2 * i + k];
            c.s.prev[2 * i + k] = p0;
            const double nw = p0 + c.s.force[2 * i + k] * dt + z[k] * scale;
            const double w = wrap1(nw, L);
            const long long ci = (long long)rint((nw - w) / L);
            pos[2 * i + k] = w;
            c.w.cross8[2 * i + k] = (int8_t)ci;
            if (cross64) cross64[2 * i + k] = (int64_t)ci;
            if (c.s.image) c.s.image[2 * i + k] += (int32_t)ci;
            crossed |= ci != 0;
        }
        R.add((u64)crossed);
    }
    return R.close(r);
}

// apply_crossings (triangulation.py:166-177), only called when some particle crossed
template <class X>
BD_HD void ph_apply_crossings(X& x, Ctx& c) {
    c.work[WK_APPLY_CROSS]++;
    bd_tri_t& T = c.s.tri;
    for (int64_t t = x.tid(); t < T.nt; t += x.nth()) {
        int32_t ts[3][2];
        for (int k = 0; k < 3; ++k)
            for (int q = 0; q < 2; ++q)
                ts[k][q] = (int32_t)T.tri_shift[6 * t + 2 * k + q] + (int32_t)c.w.cross8[2 * (int64_t)T.tri_v[3 * t + k] + q];
        for (int k = 0; k < 3; ++k)
            for (int q = 0; q < 2; ++q) T.tri_shift[6 * t + 2 * k + q] = (int8_t)(ts[k][q] - ts[0][q]);
    }
    x.sync();
}

// edge_inversion_present (triangulation.py:240-250)
template <class X>
BD_HD bool ph_edge_inversion(X& x, Red<X>& R, Ctx& c) {
    c.work[WK_EDGE_INV]++;
    u64* r = R.open();
    const bd_tri_t& T = c.s.tri;
    const double* prev = c.s.prev;
    const double* cur = c.s.pos;
    for (int64_t e = x.tid(); e < T.ne; e += x.nth()) {
        const int64_t a = T.edge_v[2 * e], b = T.edge_v[2 * e + 1];
        const double d0x = mi_exact(prev[2 * b] - prev[2 * a], c.p), d0y = mi_exact(prev[2 * b + 1] - prev[2 * a + 1], c.p);
        const double d1x = mi_exact(cur[2 * b] - cur[2 * a], c.p), d1y = mi_exact(cur[2 * b + 1] - cur[2 * a + 1], c.p);
        R.add((u64)(d0x * d1x + d0y * d1y < 0.0));
    }
    return R.close(r) != 0;
}

// signed_area2 <= 0 per triangle (into w.tinv), added to the open reduction
template <class X>
BD_HD void inverted_tris_body(X& x, Red<X>& R, Ctx& c, int shift) {
    const bd_tri_t& T = c.s.tri;
    for (int64_t t = x.tid(); t < T.nt; t += x.nth()) {
        V2 xy[3];
        tri_xy(T, c.s.pos, c.p.L, t, xy);
        const double e1x = xy[1].x - xy[0].x, e1y = xy[1].y - xy[0].y;
        const double e2x = xy[2].x - xy[0].x, e2y = xy[2].y - xy[0].y;
        const bool inv = e1x * e2y - e1y * e2x <= 0.0;
        c.w.tinv[t] = (uint8_t)inv;
        R.add((u64)inv << shift);
    }
}

// signed_area2 <= 0 per triangle; returns #inverted
template <class X>
BD_HD u64 ph_inverted_tris(X& x, Red<X>& R, Ctx& c) {
    c.work[WK_AREA_PASS]++;
    u64* r = R.open();
    inverted_tris_body(x, R, c, 0);
    return R.close(r);
}

// edge_inversion_present and the first inverted-triangle pass of
// repair_inversions in one phase (both only read positions and topology):
// low word = inverted edges, high word = inverted triangles
template <class X>
BD_HD u64 ph_edge_inversion_and_area(X& x, Red<X>& R, Ctx& c) {
    c.work[WK_EDGE_INV]++;
    c.work[WK_AREA_PASS]++;
    u64* r = R.open();
    const bd_tri_t& T = c.s.tri;
    const double* prev = c.s.prev;
    const double* cur = c.s.pos;
    for (int64_t e = x.tid(); e < T.ne; e += x.nth()) {
        const int64_t a = T.edge_v[2 * e], b = T.edge_v[2 * e + 1];
        const double d0x = mi_exact(prev[2 * b] - prev[2 * a], c.p), d0y = mi_exact(prev[2 * b + 1] - prev[2 * a + 1], c.p);
        const double d1x = mi_exact(cur[2 * b] - cur[2 * a], c.p), d1y = mi_exact(cur[2 * b + 1] - cur[2 * a + 1], c.p);
        R.add((u64)(d0x * d1x + d0y * d1y < 0.0));
    }
    inverted_tris_body(x, R, c, 32);
    return R.close(r);
}

// lexicographically-first maximal independent set of the flagged edges
// (== the reference's greedy ascending scan, triangulation.py:304-315),
// then the flips of the selected edges.  Returns #flips.  The flagged edges
// are list[0..m) when a list is given (restore_delaunay's worklist), else
// every edge with estat == ES_UND; the result does not depend on the list
// order (it is defined by the edge ids).
// dirty/gen (restore_delaunay_full): every flipped edge and the four outer
// edges of its quad -- the only edges whose quads a flip changes -- get
// dirty[.] = gen
template <class X>
BD_HD u64 ph_select_and_flip(X& x, Red<X>& R, Ctx& c, const int32_t* list = nullptr, int64_t m = 0,
                             uint32_t* dirty = nullptr, uint32_t gen = 0) {
    bd_tri_t& T = c.s.tri;
    uint8_t* st = c.w.estat;
    uint32_t* ewin = c.w.ewin;
    const int64_t cnt = list ? m : T.ne;
    u64 nsel_total = 0;
    // Round r marks its winners with stamp s0 + r in ewin (never read in the
    // phase that writes it); the states in st change only in the second
    // phase, where every thread writes its own edges and reads only ewin.
    // No read races a write: compute-sanitizer racecheck clean.  Stamps of
    // earlier calls are < s0 (a monotone counter in the control block).
    const uint32_t s0 = (uint32_t)x.ld(&c.w.ctl->wgen) + 1;
    uint32_t stamp = s0;
    for (;; ++stamp) {
        c.work[WK_LFMIS_ROUND]++;
        // an undecided edge wins when no lower-id edge of its two triangles is undecided or selected
        u64* rs = R.open();
        for (int64_t j = x.tid(); j < cnt; j += x.nth()) {
            const int64_t e = list ? list[j] : j;
            if (st[e] != ES_UND) continue;
            bool win = true;
            for (int side = 0; side < 2 && win; ++side) {
                const int64_t t = T.edge_tri[2 * e + side];
                for (int k = 0; k < 3; ++k) {
                    const int64_t f = T.tri_edge[3 * t + k];
                    if (f < e) {
                        const uint8_t sf = st[f];
                        if (sf == ES_UND || sf == ES_SEL) {
                            win = false;
                            break;
                        }
                    }
                }
            }
            if (win) ewin[e] = stamp;
            R.add((u64)win);
        }
        nsel_total += R.close(rs);
        // winners -> selected; an undecided edge next to an edge selected in this call -> removed
        u64* ru = R.open();
        for (int64_t j = x.tid(); j < cnt; j += x.nth()) {
            const int64_t e = list ? list[j] : j;
            if (st[e] != ES_UND) continue;
            if (ewin[e] == stamp) {
                st[e] = ES_SEL;
                continue;
            }
            bool blocked = false;
            for (int side = 0; side < 2 && !blocked; ++side) {
                const int64_t t = T.edge_tri[2 * e + side];
                for (int k = 0; k < 3; ++k) {
                    const int64_t f = T.tri_edge[3 * t + k];
                    if (f != e && ewin[f] >= s0 && ewin[f] <= stamp) {
                        blocked = true;
                        break;
                    }
                }
            }
            if (blocked) st[e] = ES_REM;
            R.add((u64)!blocked);
        }
        if (R.close(ru) == 0) break;
    }
    if (x.leader()) c.w.ctl->wgen = stamp;  // read again only after the flip phase's barrier
    if (nsel_total == 0) return 0;
    c.work[WK_FLIPS] += (int64_t)nsel_total;
    for (int64_t j = x.tid(); j < cnt; j += x.nth()) {
        const int64_t e = list ? list[j] : j;
        if (st[e] != ES_SEL) continue;
        const int rc = flip_edge(T, e);
        if (rc) set_error(x, c, (u64)rc, e, 0);
        if (dirty) {  // this flip's two triangles are touched by no other flip of the round
            dirty[e] = gen;
            for (int side = 0; side < 2; ++side) {
                const int64_t t = T.edge_tri[2 * e + side];
                for (int k = 0; k < 3; ++k) dirty[T.tri_edge[3 * t + k]] = gen;
            }
        }
    }
    x.sync();
    return nsel_total;
}

// in-circle flag of edge e into estat; appends flagged edges to `out`
template <class X>
BD_HD bool flag_edge(X& x, Ctx& c, int64_t e, int32_t* out, u64* out_len) {
    V2 q[4];
    edge_quad(c.s.tri, c.s.pos, c.p.L, e, q);
    const bool f = incircle(q[0], q[1], q[2], q[3], c.p.tol);
    c.w.estat[e] = f ? ES_UND : ES_NONE;
    if (f) out[x.append(out_len)] = (int32_t)e;
    return f;
}

// restore_delaunay (triangulation.py:319-334); returns passes, or -1 on error.
// The reference re-flags every edge each pass.  Positions do not move while
// it runs, so after the first pass only the edges a flip can have changed
// are re-evaluated: the flagged edges (flipped or not) and the boundary
// edges of the flipped quads; every other edge keeps its (clear) flag.  The
// per-pass flags, the flips and the pass count are the reference's.
// worklist passes cost two extra grid barriers per pass: below this many
// edges the barriers dominate and every pass re-flags all edges instead
// (cfg3: 0.79 vs 0.84 ms per step; cfg4, 3.1M edges: 3.71 vs 3.81 ms).
// BD_WORKLIST_MIN_EDGES overrides (tests run both variants on the goldens).
constexpr int64_t WORKLIST_MIN_EDGES = 1 << 20;
#if defined(__CUDACC__)
__device__ int64_t d_wl_min_edges = WORKLIST_MIN_EDGES;
#endif
BD_HD int64_t wl_min_edges() {
#if defined(__CUDA_ARCH__)
    return d_wl_min_edges;
#else
    const char* e = getenv("BD_WORKLIST_MIN_EDGES");  // host emulation: read per call
    return e ? atoll(e) : WORKLIST_MIN_EDGES;
#endif
}

// Every pass re-flags every edge, but after the first only the edges a flip
// touched (stamped by ph_select_and_flip) are re-tested: positions do not
// move inside restore_delaunay, so every other edge keeps its quad and its
// flag (flagged edges that were not flipped are ES_REM after selection).
// Same flags, flips and pass counts as re-testing everything; no extra
// barrier.
template <class X>
BD_HD int64_t restore_delaunay_full(X& x, Red<X>& R, Ctx& c, int64_t max_passes) {
    bd_tri_t& T = c.s.tri;
    const u64 gen0 = x.ld(&c.w.ctl->gen);  // stamps of this call: gen0 + 1, gen0 + 2, ...
    int64_t passes = 0;
    for (;;) {
        c.work[WK_FLAG_PASS]++;
        const uint32_t gen = (uint32_t)(gen0 + (u64)passes);
        u64* r = R.open();
        for (int64_t e = x.tid(); e < T.ne; e += x.nth()) {
            bool f;
            if (passes == 0 || c.w.stamp[e] == gen) {
                V2 q[4];
                edge_quad(T, c.s.pos, c.p.L, e, q);
                f = incircle(q[0], q[1], q[2], q[3], c.p.tol);
            } else {
                f = c.w.estat[e] != ES_NONE;
            }
            c.w.estat[e] = f ? ES_UND : ES_NONE;
            R.add((u64)f);
        }
        if (R.close(r) == 0) {
            if (x.leader()) c.w.ctl->gen = gen0 + (u64)passes + 1;  // read again only after the next call's barrier
            return passes;
        }
        passes++;
        if (passes > max_passes) {
            // error exits also retire this call's stamps (a caller may catch
            // the error and call again: its stamps must not look current)
            if (x.leader()) c.w.ctl->gen = gen0 + (u64)passes + 1;
            set_error(x, c, BD_ERR_NONCONV, passes, 0);
            x.sync();
            return -1;
        }
        ph_select_and_flip(x, R, c, nullptr, 0, c.w.stamp, (uint32_t)(gen0 + (u64)passes));
        if (x.ld(&c.w.ctl->status)) {
            if (x.leader()) c.w.ctl->gen = gen0 + (u64)passes + 1;
            return -1;
        }
    }
}

template <class X>
BD_HD int64_t restore_delaunay(X& x, Red<X>& R, Ctx& c, int64_t max_passes) {
    bd_tri_t& T = c.s.tri;
    if (T.ne < wl_min_edges()) return restore_delaunay_full(x, R, c, max_passes);
    u64* lens = c.w.ctl->lists;  // flagged-list lengths in lens[0..3], candidate lengths in lens[4..7]
    int32_t* flagged = c.w.wl0;
    int32_t* cand = c.w.wl1;
    int64_t passes = 0;
    // pass 1 over every edge
    c.work[WK_FLAG_PASS]++;
    if (x.leader()) {
        for (int k = 0; k < 8; ++k) lens[k] = 0;
    }
    x.sync();
    const u64 gen0 = x.ld(&c.w.ctl->gen);  // stamps of this call: gen0 + 1, gen0 + 2, ...
    u64* r = R.open();
    for (int64_t e = x.tid(); e < T.ne; e += x.nth()) R.add((u64)flag_edge(x, c, e, flagged, &lens[0]));
    u64 nflag = R.close(r);
    for (;;) {
        if (nflag == 0) {
            if (x.leader()) c.w.ctl->gen = gen0 + (u64)passes + 1;  // read again only after the next call's barrier
            return passes;
        }
        passes++;
        if (passes > max_passes) {
            if (x.leader()) c.w.ctl->gen = gen0 + (u64)passes + 1;  // retire this call's stamps (see above)
            set_error(x, c, BD_ERR_NONCONV, passes, 0);
            x.sync();
            return -1;
        }
        ph_select_and_flip(x, R, c, flagged, (int64_t)nflag);
        if (x.ld(&c.w.ctl->status)) {
            if (x.leader()) c.w.ctl->gen = gen0 + (u64)passes + 1;
            return -1;
        }
        // candidates of the next pass (deduplicated by a per-call generation stamp)
        const int ring = (int)(passes & 3);
        u64* nc = &lens[4 + ring];
        if (x.leader()) {
            lens[4 + ((ring + 1) & 3)] = 0;  // reset the next rings before anyone appends to them
            lens[(ring + 1) & 3] = 0;
        }
        const uint32_t gen = (uint32_t)(gen0 + (u64)passes);
        for (int64_t j = x.tid(); j < (int64_t)nflag; j += x.nth()) {
            const int64_t e = flagged[j];
            const bool flipped = c.w.estat[e] == ES_SEL;
            if (x.exch32(&c.w.stamp[e], gen) != gen) cand[x.append(nc)] = (int32_t)e;
            if (!flipped) continue;
            for (int side = 0; side < 2; ++side) {
                const int64_t t = T.edge_tri[2 * e + side];
                for (int k = 0; k < 3; ++k) {
                    const int64_t f = T.tri_edge[3 * t + k];
                    if (f != e && x.exch32(&c.w.stamp[f], gen) != gen) cand[x.append(nc)] = (int32_t)f;
                }
            }
        }
        x.sync();
        const int64_t ncand = (int64_t)x.ld(nc);
        // re-evaluate the candidates into the flagged list of the next pass
        c.work[WK_FLAG_EDGES_WL] += ncand;
        u64* nf = &lens[(ring + 1) & 3];
        r = R.open();
        for (int64_t j = x.tid(); j < ncand; j += x.nth()) R.add((u64)flag_edge(x, c, cand[j], flagged, nf));
        nflag = R.close(r);
    }
}

// repair_inversions (triangulation.py:336-363) with prev = positions_prev
// (use_prev = false: the reference's prev=None, local predicate only).
// returns 0 ok, 1 needs rollback, -1 error; adds flips to *flips and, if
// given, the reference's RepairResult.passes to *passes
template <class X>
BD_HD int repair_inversions(X& x, Red<X>& R, Ctx& c, int64_t max_passes, int64_t* flips, bool use_prev = true,
                            int64_t* passes = nullptr, int64_t inverted0 = -1) {
    bd_tri_t& T = c.s.tri;
    for (int64_t pass = 0; pass < max_passes; ++pass) {
        if (passes) *passes = pass;
        // inverted0: the first pass's count (and w.tinv) already computed by the caller
        const u64 ninv = pass == 0 && inverted0 >= 0 ? (u64)inverted0 : ph_inverted_tris(x, R, c);
        if (ninv == 0) return 0;
        c.work[WK_FLAG_PASS]++;
        for (int64_t e = x.tid(); e < T.ne; e += x.nth()) {
            V2 q[4];
            edge_quad(T, c.s.pos, c.p.L, e, q);
            bool f = point_in_tri(q[3], q[0], q[1], q[2]) | point_in_tri(q[2], q[0], q[1], q[3]);
            for (int side = 0; side < 2 && !f && use_prev; ++side) {
                const int64_t t = T.edge_tri[2 * e + side];
                if (c.w.tinv[t]) f = crossed_side(T, c.s.pos, c.s.prev, c.p, t, T.edge_opp[2 * e + side]);
            }
            c.w.estat[e] = f ? ES_UND : ES_NONE;
        }
        x.sync();
        const u64 chosen = ph_select_and_flip(x, R, c);
        if (x.ld(&c.w.ctl->status)) return -1;
        if (chosen == 0) return 1;
        *flips += (int64_t)chosen;
    }
    if (passes) *passes = max_passes;
    return ph_inverted_tris(x, R, c) != 0 ? 1 : 0;
}

// edge_inversion_present + repair_inversions + restore_delaunay
// (dynamics.py:206-214 and :236-242): 0 ok, 1 rollback, -1 error
template <class X>
BD_HD int maintain(X& x, Red<X>& R, Ctx& c, int64_t* repairs, int64_t* flip_passes) {
    const u64 v = ph_edge_inversion_and_area(x, R, c);
    if (v & 0xffffffffull) return 1;
    const int rr = repair_inversions(x, R, c, 10, repairs, true, nullptr, (int64_t)(v >> 32));
    if (rr) return rr;
    const int64_t p = restore_delaunay(x, R, c, 1000);
    if (p < 0) return -1;
    *flip_passes += p;
    return 0;
}

// Pair sources for the overlap correction / incidence lists: the
// triangulation edges (dynamics.py:226-229), every Verlet pair, or the
// Verlet overlap-candidate subset (forces.py:145-149).
struct EdgePairs {
    const int32_t* ev;
    int64_t m;
    BD_HD int64_t count() const { return m; }
    BD_HD int64_t a(int64_t e) const { return ev[2 * e]; }
    BD_HD int64_t b(int64_t e) const { return ev[2 * e + 1]; }
};

struct ListPairs {
    const int64_t* pa;
    const int64_t* pb;
    int64_t m;
    BD_HD int64_t count() const { return m; }
    BD_HD int64_t a(int64_t e) const { return pa[e]; }
    BD_HD int64_t b(int64_t e) const { return pb[e]; }
};

struct SubsetPairs {
    const int64_t* pa;
    const int64_t* pb;
    const int32_t* idx;
    int64_t m;
    BD_HD int64_t count() const { return m; }
    BD_HD int64_t a(int64_t e) const { return pa[idx[e]]; }
    BD_HD int64_t b(int64_t e) const { return pb[idx[e]]; }
};

// vertex -> incident pairs, ascending pair index (fixes the reference's
// ascending-pair accumulation order of overlap_pass_kernel / short_range_kernel)
template <class X, class PS>
BD_HD void build_incidence(X& x, int64_t n, const PS& ps, int32_t* off, int32_t* cur, int32_t* inc,
                           int64_t* work = nullptr) {
    if (work) work[WK_INCIDENCE]++;
    for (int64_t i = x.tid(); i < n; i += x.nth()) {
        off[i] = 0;
        cur[i] = 0;
    }
    x.sync();
    const int64_t m = ps.count();
    for (int64_t e = x.tid(); e < m; e += x.nth()) {
        x.fetch_add32(&off[ps.a(e)], 1);
        x.fetch_add32(&off[ps.b(e)], 1);
    }
    x.sync();
    x.exclusive_scan(off, n);
    for (int64_t e = x.tid(); e < m; e += x.nth()) {
        const int64_t a = ps.a(e), b = ps.b(e);
        inc[off[a] + x.fetch_add32(&cur[a], 1)] = (int32_t)e;
        inc[off[b] + x.fetch_add32(&cur[b], 1)] = (int32_t)e;
    }
    x.sync();
    for (int64_t i = x.tid(); i < n; i += x.nth()) {
        int32_t* Lst = inc + off[i];
        const int32_t k = off[i + 1] - off[i];
        if (k <= 16) {  // the usual case (Delaunay degree ~6): sort a private copy, one pass in, one out
            int32_t v[16];
            for (int32_t j = 0; j < k; ++j) v[j] = Lst[j];
            for (int32_t j = 1; j < k; ++j) {
                const int32_t t = v[j];
                int32_t q = j - 1;
                while (q >= 0 && v[q] > t) {
                    v[q + 1] = v[q];
                    --q;
                }
                v[q + 1] = t;
            }
            for (int32_t j = 0; j < k; ++j) Lst[j] = v[j];
            continue;
        }
        for (int32_t j = 1; j < k; ++j) {
            const int32_t t = Lst[j];
            int32_t q = j - 1;
            while (q >= 0 && Lst[q] > t) {
                Lst[q + 1] = Lst[q];
                --q;
            }
            Lst[q + 1] = t;
        }
    }
    x.sync();
}

template <class X>
BD_HD void build_edge_incidence(X& x, Ctx& c) {
    const EdgePairs ps{c.s.tri.edge_v, c.s.tri.ne};
    build_incidence(x, c.p.n, ps, c.w.inc_off, c.w.inc_cur, c.w.inc, c.work);
}

// the edge incidence lists when stale: they depend on edge_v only, which
// only flips (and a rollback) change
template <class X>
BD_HD void build_edge_incidence_t(X& x, Ctx& c) {
    if (c.inc_flips == c.work[WK_FLIPS]) return;
    const int64_t t0 = now_ns();
    build_edge_incidence(x, c);
    c.inc_flips = c.work[WK_FLIPS];
    c.work[WK_T_INCIDENCE] += now_ns() - t0;
}

// correct_overlaps (dynamics.py:97-133) over a fixed pair set with its
// incidence lists in w.inc_off / w.inc; `tri` -> crossings feed
// apply_crossings (dynamics.py:127-129).  Returns sweeps, -1 on non-convergence.
// edge_inc: ps are the triangulation edges and their incidence lists are
// built here, only once a pass finds an overlap (most calls after a
// maintenance round find none and never need them)
template <class X, class PS>
BD_HD int64_t correct_overlaps(X& x, Red<X>& R, Ctx& c, const PS& ps, bool tri, bool edge_inc = false) {
    const double L = c.p.L, sigma = c.p.sigma, thresh = sigma * (1.0 - 1e-9), cap = c.p.cap;
    double* pos = c.s.pos;
    const int64_t m = ps.count();
    int64_t iterations = 0;
    // particles with an overlapping pair are stamped in the pass, so the
    // apply gathers only theirs (the rest just clear their crossings)
    const u64 g0 = x.ld(&c.w.ctl->vgen);
    for (int64_t it = 0; it < c.p.max_overlap_iters; ++it) {
        c.work[WK_OVL_PASS]++;
        const uint32_t gen = (uint32_t)(g0 + 1 + (u64)it);
        u64* r = R.open();
        for (int64_t e = x.tid(); e < m; e += x.nth()) {
            const int64_t a = ps.a(e), b = ps.b(e);
            const double dx = mi_exact(pos[2 * b] - pos[2 * a], c.p), dy = mi_exact(pos[2 * b + 1] - pos[2 * a + 1], c.p);
            const double rr = sqrt(dx * dx + dy * dy);
            const bool ov = !(rr >= thresh || rr == 0.0);
            if (ov) {
                const double delta = sigma - rr;
                const double ux = dx / rr, uy = dy / rr;
                c.w.contrib[2 * e] = delta * ux;
                c.w.contrib[2 * e + 1] = delta * uy;
                c.w.vhit[a] = gen;
                c.w.vhit[b] = gen;
            }
            c.w.eovl[e] = (uint8_t)ov;
            R.add((u64)ov);
        }
        if (R.close(r) == 0) {
            if (x.leader()) c.w.ctl->vgen = g0 + 2 + (u64)it;  // read again after the next call's barrier
            return iterations;
        }
        iterations++;
        if (edge_inc) build_edge_incidence_t(x, c);
        c.work[WK_OVL_APPLY]++;
        u64* rc = R.open();
        for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) {
            if (c.w.vhit[i] != gen) {
                c.w.cross8[2 * i] = 0;
                c.w.cross8[2 * i + 1] = 0;
                continue;
            }
            double dx = 0.0, dy = 0.0;
            bool hit = false;
            const int32_t j0 = c.w.inc_off[i], j1 = c.w.inc_off[i + 1];
            for (int32_t j = j0; j < j1; ++j) {
                const int64_t e = c.w.inc[j];
                if (!c.w.eovl[e]) continue;
                hit = true;
                const double cx = c.w.contrib[2 * e], cy = c.w.contrib[2 * e + 1];
                if (ps.a(e) == i) {
                    dx -= cx;
                    dy -= cy;
                } else {
                    dx += cx;
                    dy += cy;
                }
            }
            int crossed = 0;
            if (hit) {
                c.s.overlap_flags[i] = 1;
                const double norm = sqrt(dx * dx + dy * dy);
                double factor = 1.0;
                if (norm > cap) factor = cap / norm;
                const double d[2] = {dx, dy};
                for (int k = 0; k < 2; ++k) {
                    const double nw = pos[2 * i + k] + d[k] * factor;
                    const double w = wrap1(nw, L);
                    const long long ci = (long long)rint((nw - w) / L);
                    pos[2 * i + k] = w;
                    c.w.cross8[2 * i + k] = (int8_t)ci;
                    if (c.s.image) c.s.image[2 * i + k] += (int32_t)ci;
                    crossed |= ci != 0;
                }
            } else {
                c.w.cross8[2 * i] = 0;
                c.w.cross8[2 * i + 1] = 0;
            }
            R.add((u64)crossed);
        }
        if (R.close(rc) && tri) ph_apply_crossings(x, c);
    }
    if (x.leader()) c.w.ctl->vgen = g0 + 2 + (u64)c.p.max_overlap_iters;
    set_error(x, c, BD_ERR_NONCONV, 0, 0);
    x.sync();
    return -1;
}

}  // namespace bd
