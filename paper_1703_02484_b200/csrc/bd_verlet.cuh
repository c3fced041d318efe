// bd_verlet.cuh -- short-range force path on the device: Verlet list build
// (cell grid + ordered pair emission), staleness test, short-range forces,
// overlap-candidate subset.  Same uniform-phase style as bd_step.cuh.
//
// Reference: build_cell_grid forces.py:81-99, _kernels.cell_pairs
// _kernels.py:141-236, build_verlet forces.py:120-150, verlet_needs_rebuild
// forces.py:153-156 (max_sq_displacement _kernels.py:128-138),
// short_range_kernel _kernels.py:62-91.
//
// Bit-exactness: the pair list has exactly the reference's order (cells
// ascending; same cell ia < ib in stable cell order; half-neighbourhood
// offsets (1,0), (-1,1), (0,1), (1,1); a in c x b in d), produced by one
// thread per cell in two passes (count, fill) around a scan.  Short-range
// forces are gathered per particle over its incident pairs in ascending pair
// index, reproducing the reference's sequential += / -= order.
#pragma once

#include "bd_step.cuh"

namespace bd {

// half-neighbourhood offsets (1,0), (-1,1), (0,1), (1,1) (_kernels.py:159-167)
BD_HD int off_x(int k) { return k == 0 ? 1 : (k == 1 ? -1 : (k == 2 ? 0 : 1)); }
BD_HD int off_y(int k) { return k == 0 ? 0 : 1; }

// The reference emits the pairs of cell c (ascending c) in the order
//   segment 0: same cell, ia < ib;  segments 1..4: neighbour offsets
//   (1,0), (-1,1), (0,1), (1,1), a in c x b in d   (_kernels.py:141-236),
// a ascending inside every segment.  One work item per (cell, segment, a):
// its pairs are contiguous in that order, so items are counted, scanned in
// (cell, segment, a) order and filled independently -- 5 N short items
// instead of one long sequential walk per cell.  Item index of sorted slot
// s (particle corder[s] in cell c, local index s - start_c) and segment g:
//   5 start_c + g m_c + (s - start_c),   m_c = particles in c.
BD_HD int64_t vl_item(const Ctx& c, int64_t s, int g, int64_t* cell, int64_t* ia) {
    const int64_t a = c.w.corder[s];
    const int64_t cc = c.w.cell_id[a];
    const int64_t st = c.w.cell_start[cc], m = c.w.cell_start[cc + 1] - st;
    *cell = cc;
    *ia = s - st;
    return 5 * st + (int64_t)g * m + (s - st);
}

template <bool FILL>
BD_HD int64_t item_pairs_of(const Ctx& c, int64_t cell, int64_t ia, int g, int64_t k0) {
    const int64_t ncx = c.p.ncx;
    const int64_t cx = cell % ncx, cy = cell / ncx;
    const int32_t a0 = c.w.cell_start[cell];
    const double rl2 = c.p.r_list * c.p.r_list;
    const double* pos = c.s.pos;
    const int64_t a = c.w.corder[a0 + ia];
    const double xa = pos[2 * a], ya = pos[2 * a + 1];
    int32_t b0, b1;
    if (g == 0) {
        b0 = a0 + (int32_t)ia + 1;
        b1 = c.w.cell_start[cell + 1];
    } else {
        const int64_t d = ((cx + off_x(g - 1) + ncx) % ncx) + ((cy + off_y(g - 1)) % ncx) * ncx;
        b0 = c.w.cell_start[d];
        b1 = c.w.cell_start[d + 1];
    }
    int64_t k = k0;
    for (int32_t ib = b0; ib < b1; ++ib) {
        const int64_t b = c.w.corder[ib];
        const double dx = mi_exact(xa - pos[2 * b], c.p), dy = mi_exact(ya - pos[2 * b + 1], c.p);
        if (dx * dx + dy * dy <= rl2) {
            if (FILL) {
                c.s.pair_a[k] = a;
                c.s.pair_b[k] = b;
            }
            ++k;
        }
    }
    return k - k0;
}

// one row a of np.triu_indices(n, 1) within r_list (forces.py:136-141, no grid)
template <bool FILL>
BD_HD int64_t brute_pairs_of(const Ctx& c, int64_t a, int64_t k0) {
    const double rl2 = c.p.r_list * c.p.r_list;
    const double* pos = c.s.pos;
    int64_t k = k0;
    for (int64_t b = a + 1; b < c.p.n; ++b) {
        const double dx = mi_exact(pos[2 * b] - pos[2 * a], c.p), dy = mi_exact(pos[2 * b + 1] - pos[2 * a + 1], c.p);
        if (dx * dx + dy * dy <= rl2) {
            if (FILL) {
                c.s.pair_a[k] = a;
                c.s.pair_b[k] = b;
            }
            ++k;
        }
    }
    return k - k0;
}

// verlet_needs_rebuild: never built, or max |mi(pos - snap)|^2 > (skin/2)^2
template <class X>
BD_HD bool vl_stale(X& x, Red<X>& R, Ctx& c) {
    if (x.ld((const u64*)&c.s.vl_meta[1]) == 0) return true;
    u64* r = R.open();
    u64 m = 0;  // d2 >= 0: its bit pattern orders like the value
    for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) {
        const double dx = mi_exact(c.s.pos[2 * i] - c.s.vl_snap[2 * i], c.p);
        const double dy = mi_exact(c.s.pos[2 * i + 1] - c.s.vl_snap[2 * i + 1], c.p);
        const u64 b = double_to_bits(dx * dx + dy * dy);
        m = b > m ? b : m;
    }
    x.umax_all(r, m);  // one atomic per warp, not per particle
    const double worst = bits_to_double(R.close(r));
    const double h = c.p.skin / 2.0;
    return worst > h * h;
}

// build_cell_grid + cell_pairs + snapshot (+ overlap subset within `margin`
// when margin > 0, + the per-particle pair incidence for the force gather).
// Returns false on a capacity overflow (status BD_ERR_CAPACITY).
template <class X>
BD_HD bool vl_rebuild_impl(X& x, Red<X>& R, Ctx& c, double margin);

template <class X>
BD_HD bool vl_rebuild(X& x, Red<X>& R, Ctx& c, double margin) {
    const int64_t t0 = now_ns();
    const bool ok = vl_rebuild_impl(x, R, c, margin);
    c.work[WK_T_VERLET] += now_ns() - t0;
    return ok;
}

template <class X>
BD_HD bool vl_rebuild_impl(X& x, Red<X>& R, Ctx& c, double margin) {
    c.work[WK_VL_REBUILD]++;
    const int64_t n = c.p.n, ncx = c.p.ncx;
    int32_t* cnt = c.w.pcnt;
    int64_t rows;
    if (ncx >= 3) {
        const int64_t nc = ncx * ncx;
        const double edge = c.p.L / (double)ncx;
        for (int64_t k = x.tid(); k < nc; k += x.nth()) {
            c.w.cell_start[k] = 0;
            c.w.cell_cur[k] = 0;
        }
        x.sync();
        for (int64_t i = x.tid(); i < n; i += x.nth()) {
            int64_t ix = (int64_t)floor(c.s.pos[2 * i] / edge), iy = (int64_t)floor(c.s.pos[2 * i + 1] / edge);
            ix = ix < 0 ? 0 : (ix > ncx - 1 ? ncx - 1 : ix);
            iy = iy < 0 ? 0 : (iy > ncx - 1 ? ncx - 1 : iy);
            const int32_t cid = (int32_t)(ix + iy * ncx);
            c.w.cell_id[i] = cid;
            x.fetch_add32(&c.w.cell_start[cid], 1);
        }
        x.sync();
        x.exclusive_scan(c.w.cell_start, nc);
        for (int64_t i = x.tid(); i < n; i += x.nth()) {
            const int32_t cid = c.w.cell_id[i];
            c.w.corder[c.w.cell_start[cid] + x.fetch_add32(&c.w.cell_cur[cid], 1)] = (int32_t)i;
        }
        x.sync();
        // stable argsort: ascending particle index inside each cell
        for (int64_t k = x.tid(); k < nc; k += x.nth()) {
            int32_t* a = c.w.corder + c.w.cell_start[k];
            const int32_t m = c.w.cell_start[k + 1] - c.w.cell_start[k];
            if (m <= 24) {  // the usual case: sort a private copy (one pass in, one out)
                int32_t v[24];
                for (int32_t j = 0; j < m; ++j) v[j] = a[j];
                for (int32_t j = 1; j < m; ++j) {
                    const int32_t t = v[j];
                    int32_t q = j - 1;
                    while (q >= 0 && v[q] > t) {
                        v[q + 1] = v[q];
                        --q;
                    }
                    v[q + 1] = t;
                }
                for (int32_t j = 0; j < m; ++j) a[j] = v[j];
                continue;
            }
            for (int32_t j = 1; j < m; ++j) {
                const int32_t v = a[j];
                int32_t q = j - 1;
                while (q >= 0 && a[q] > v) {
                    a[q + 1] = a[q];
                    --q;
                }
                a[q + 1] = v;
            }
        }
        x.sync();
        for (int64_t t = x.tid(); t < 5 * n; t += x.nth()) {
            const int64_t sl = t / 5;
            const int g = (int)(t % 5);
            int64_t cell, ia;
            const int64_t item = vl_item(c, sl, g, &cell, &ia);
            cnt[item] = (int32_t)item_pairs_of<false>(c, cell, ia, g, 0);
        }
        rows = 5 * n;
    } else {
        for (int64_t a = x.tid(); a < n; a += x.nth()) cnt[a] = (int32_t)brute_pairs_of<false>(c, a, 0);
        rows = n;
    }
    x.sync();
    x.exclusive_scan(cnt, rows);
    const int64_t total = cnt[rows];
    if (total > c.p.pair_capacity) {
        set_error(x, c, BD_ERR_CAPACITY, total, c.p.pair_capacity);
        x.sync();
        return false;
    }
    if (ncx >= 3)
        for (int64_t t = x.tid(); t < 5 * n; t += x.nth()) {
            const int64_t sl = t / 5;
            const int g = (int)(t % 5);
            int64_t cell, ia;
            const int64_t item = vl_item(c, sl, g, &cell, &ia);
            item_pairs_of<true>(c, cell, ia, g, cnt[item]);
        }
    else
        for (int64_t a = x.tid(); a < rows; a += x.nth()) brute_pairs_of<true>(c, a, cnt[a]);
    for (int64_t i = x.tid(); i < 2 * n; i += x.nth()) c.s.vl_snap[i] = c.s.pos[i];
    x.sync();
    // incidence of the Verlet pairs (ascending pair index per particle)
    const ListPairs lp{c.s.pair_a, c.s.pair_b, total};
    build_incidence(x, n, lp, c.w.vinc_off, c.w.vinc_cur, c.w.vinc, c.work);
    int64_t nov = 0;
    if (margin > 0.0) {
        // overlap candidates: pairs within margin at build time, order kept (forces.py:145-149)
        int32_t* flag = (int32_t*)c.w.contrib;  // scratch (>= 4 (P+1) bytes)
        const double m2 = margin * margin;
        for (int64_t e = x.tid(); e < total; e += x.nth()) {
            const int64_t a = c.s.pair_a[e], b = c.s.pair_b[e];
            const double dx = mi_exact(c.s.pos[2 * b] - c.s.pos[2 * a], c.p);
            const double dy = mi_exact(c.s.pos[2 * b + 1] - c.s.pos[2 * a + 1], c.p);
            flag[e] = (dx * dx + dy * dy) <= m2 ? 1 : 0;
        }
        x.sync();
        x.exclusive_scan(flag, total);
        nov = flag[total];
        for (int64_t e = x.tid(); e < total; e += x.nth())
            if (flag[e + 1] != flag[e]) c.w.ov_idx[flag[e]] = (int32_t)e;
        x.sync();
    }
    if (x.leader()) {
        c.s.vl_meta[0] = total;
        c.s.vl_meta[1] = 1;
        c.s.vl_meta[2] += 1;
        c.s.vl_meta[3] = nov;
    }
    x.sync();
    return true;
}

// short_range_kernel (_kernels.py:62-91) gathered per particle: out[i], err[i]
template <class X>
BD_HD void sr_forces_impl(X& x, Ctx& c, double* out, int64_t* err);

template <class X>
BD_HD void sr_forces(X& x, Ctx& c, double* out, int64_t* err) {
    const int64_t t0 = now_ns();
    sr_forces_impl(x, c, out, err);
    c.work[WK_T_SR_FORCE] += now_ns() - t0;
}

template <class X>
BD_HD void sr_forces_impl(X& x, Ctx& c, double* out, int64_t* err) {
    c.work[WK_SR_FORCE]++;
    const double rc2 = c.p.r_cut * c.p.r_cut;
    const double* pos = c.s.pos;
    for (int64_t i = x.tid(); i < c.p.n; i += x.nth()) {
        double fx = 0.0, fy = 0.0;
        int64_t e = 0;
        const int32_t j0 = c.w.vinc_off[i], j1 = c.w.vinc_off[i + 1];
        for (int32_t j = j0; j < j1; ++j) {
            const int64_t q = c.w.vinc[j];
            const int64_t a = c.s.pair_a[q], b = c.s.pair_b[q];
            const double dx = mi_exact(pos[2 * a] - pos[2 * b], c.p), dy = mi_exact(pos[2 * a + 1] - pos[2 * b + 1], c.p);
            const double r2 = dx * dx + dy * dy;
            if (r2 > rc2) continue;
            if (r2 == 0.0) {
                if (a == i) e = b + 1;
                continue;
            }
            const double inv7 = 1.0 / (r2 * r2 * r2 * sqrt(r2));
            if (a == i) {
                const double wa = c.s.mu[a] * c.s.alpha[b] * inv7;
                fx += wa * dx;
                fy += wa * dy;
            } else {
                const double wb = c.s.mu[b] * c.s.alpha[a] * inv7;
                fx -= wb * dx;
                fy -= wb * dy;
            }
        }
        out[2 * i] = fx;
        out[2 * i + 1] = fy;
        err[i] = e;
    }
    x.sync();
}

}  // namespace bd
