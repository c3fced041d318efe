// bd_build.cuh -- the initial periodic Delaunay triangulation, on the device.
//
// Reference: build_initial / _build_from_tiling (triangulation.py:514-648):
// jitter the points by 1e-9 L (fixed Philox key), run a planar Qhull
// Delaunay on 9 (25, 49) periodic copies, keep the triangles touching the
// fundamental domain, deduplicate them, then restore_delaunay on the
// unjittered points and audit.  It is host-serial (23.5 s at N = 131k,
// 321 s / 7.2 GB at N = 1M) and fails for cfg4's seed 0.
//
// The device build computes the same triangulation from the dual side: the
// periodic Voronoi cell of every (jittered) point, independently, by
// clipping a square against the bisectors of its neighbours in a cell grid
// -- ring by ring until the security radius proves the cell final.  The
// cell's edges, in counter-clockwise order, are the point's Delaunay
// neighbours (its "star"); consecutive neighbours close a triangle.  All
// geometry is in coordinates relative to the point (magnitudes ~ the
// spacing), so the jitter's 1e-9 L separates near-cocircular sets by ~1e-6
// of the spacing against ~1e-16 of rounding: the same decisions Qhull
// takes on the same jittered points, i.e. the same edge set.
//
// Indexing differs from the reference's (which follows Qhull's facet
// order): triangle t is owned by its smallest vertex, which sits in slot 0
// with shift (0,0); triangles and edges are numbered by owner, then by the
// owner's star position (star rotated to start at its smallest neighbour).
// Every star relation is checked from both ends (symmetry, triangle
// closure) and the counts against Euler (F = 2V, E = 3V); a failure is
// reported, never patched.  The caller then runs restore_delaunay on the
// unjittered points and the audit, exactly as the reference does.
#pragma once

#include "bd_exec.cuh"

namespace bd {

constexpr int BLD_MAXD = 32;  // star capacity (Delaunay degree) per vertex
constexpr int BLD_MAXV = 64;  // polygon capacity while clipping

// failure reasons (result[2])
enum {
    BLD_COINCIDENT = 1,
    BLD_POLY_OVERFLOW = 2,
    BLD_TOO_SPARSE = 3,
    BLD_DEGREE_OVERFLOW = 4,
    BLD_SHIFT_RANGE = 5,
    BLD_ASYMMETRIC = 6,
    BLD_INCONSISTENT = 7,
    BLD_REPEATED_VERTEX = 8,
    BLD_EULER = 9,
};

struct BuildGeo {
    int64_t n;
    double L;
    int64_t ncx;  // cells per side
    double h;     // cell edge = L / ncx
};

BD_HD BuildGeo build_geo(int64_t n, double L) {
    BuildGeo g;
    g.n = n;
    g.L = L;
    const double h0 = sqrt(2.0 * L * L / (double)(n > 0 ? n : 1));  // ~2 points per cell
    int64_t ncx = (int64_t)floor(L / h0);
    if (ncx < 1) ncx = 1;
    if (ncx > 46340) ncx = 46340;  // ncx^2 fits int32
    g.ncx = ncx;
    g.h = L / (double)ncx;
    return g;
}

struct BuildWs {
    Ctl* ctl;
    int32_t* cell_start;  // (nc+1)
    int32_t* cell_cur;    // (nc)
    int32_t* cell_pts;    // (n)
    int32_t* deg;         // (n)
    int32_t* nb;          // (n, MAXD) star: neighbour vertex, CCW
    int8_t* sh;           // (n, MAXD, 2) star: neighbour image shift
    int32_t* tcnt;        // (n+1) owned triangles -> offsets
    int32_t* ecnt;        // (n+1) owned edges -> offsets
};

struct BuildLayout {
    int64_t ctl, cell_start, cell_cur, cell_pts, deg, nb, sh, tcnt, ecnt, total;
};

BD_HD int64_t bld_align(int64_t x) { return (x + 255) & ~(int64_t)255; }

BD_HD BuildLayout build_layout(int64_t n, double L) {
    const BuildGeo g = build_geo(n, L);
    const int64_t nc = g.ncx * g.ncx;
    BuildLayout l;
    int64_t o = 0;
    l.ctl = o; o = bld_align(o + (int64_t)sizeof(Ctl));
    l.cell_start = o; o = bld_align(o + 4 * (nc + 1));
    l.cell_cur = o; o = bld_align(o + 4 * nc);
    l.cell_pts = o; o = bld_align(o + 4 * n);
    l.deg = o; o = bld_align(o + 4 * n);
    l.nb = o; o = bld_align(o + 4 * n * BLD_MAXD);
    l.sh = o; o = bld_align(o + 2 * n * BLD_MAXD);
    l.tcnt = o; o = bld_align(o + 4 * (n + 1));
    l.ecnt = o; o = bld_align(o + 4 * (n + 1));
    l.total = o;
    return l;
}

BD_HD BuildWs build_carve(void* base, int64_t n, double L) {
    const BuildLayout l = build_layout(n, L);
    char* b = (char*)base;
    BuildWs w;
    w.ctl = (Ctl*)(b + l.ctl);
    w.cell_start = (int32_t*)(b + l.cell_start);
    w.cell_cur = (int32_t*)(b + l.cell_cur);
    w.cell_pts = (int32_t*)(b + l.cell_pts);
    w.deg = (int32_t*)(b + l.deg);
    w.nb = (int32_t*)(b + l.nb);
    w.sh = (int8_t*)(b + l.sh);
    w.tcnt = (int32_t*)(b + l.tcnt);
    w.ecnt = (int32_t*)(b + l.ecnt);
    return w;
}

struct BuildCtx {
    BuildGeo g;
    BuildWs w;
    const double* pos;
    bd_tri_t out;
};

template <class X>
BD_HD void bld_fail(X& x, const BuildCtx& c, int64_t i, int64_t reason) {
    if (x.cas(&c.w.ctl->status, 0, BD_ERR_BUILD) == 0) {
        c.w.ctl->err_i = (u64)i;
        c.w.ctl->err_k = (u64)reason;
    }
}

BD_HD int64_t bld_cell_coord(double v, const BuildGeo& g) {
    const double w = v - floor(v / g.L) * g.L;
    int64_t k = (int64_t)(w / g.h);
    if (k < 0) k = 0;
    if (k >= g.ncx) k = g.ncx - 1;
    return k;
}

BD_HD int64_t bld_cell_of(const double* pos, int64_t i, const BuildGeo& g) {
    return bld_cell_coord(pos[2 * i], g) + g.ncx * bld_cell_coord(pos[2 * i + 1], g);
}

// ---- phase 1: points binned by cell, ascending index within a cell --------

template <class X>
BD_HD void bld_bin(X& x, BuildCtx& c) {
    const int64_t n = c.g.n, nc = c.g.ncx * c.g.ncx;
    for (int64_t k = x.tid(); k <= nc; k += x.nth()) c.w.cell_start[k] = 0;
    x.sync();
    for (int64_t i = x.tid(); i < n; i += x.nth()) x.fetch_add32(&c.w.cell_start[bld_cell_of(c.pos, i, c.g)], 1);
    x.sync();
    x.exclusive_scan(c.w.cell_start, nc);
    for (int64_t k = x.tid(); k < nc; k += x.nth()) c.w.cell_cur[k] = c.w.cell_start[k];
    x.sync();
    for (int64_t i = x.tid(); i < n; i += x.nth()) {
        const int32_t slot = x.fetch_add32(&c.w.cell_cur[bld_cell_of(c.pos, i, c.g)], 1);
        c.w.cell_pts[slot] = (int32_t)i;
    }
    x.sync();
    for (int64_t k = x.tid(); k < nc; k += x.nth()) {  // a handful per cell: insertion sort
        int32_t* a = c.w.cell_pts + c.w.cell_start[k];
        const int32_t m = c.w.cell_start[k + 1] - c.w.cell_start[k];
        for (int32_t u = 1; u < m; ++u) {
            const int32_t v = a[u];
            int32_t w = u - 1;
            while (w >= 0 && a[w] > v) {
                a[w + 1] = a[w];
                --w;
            }
            a[w + 1] = v;
        }
    }
    x.sync();
}

// ---- phase 2: Voronoi cell by half-plane clipping -> star -----------------

struct Poly {
    double x[BLD_MAXV], y[BLD_MAXV];
    int32_t g[BLD_MAXV];  // generator of the edge leaving vertex k (-1: initial square)
    int nv;
};

// clip by {v : v.d <= half} (the bisector of the origin and d, generator j);
// returns false on overflow.  A vertex exactly on the line stays and no
// zero-length edge is created.
BD_HD bool poly_clip(Poly& P, Poly& Q, double dx, double dy, double half, int32_t j) {
    double s[BLD_MAXV];
    bool any_out = false;
    for (int k = 0; k < P.nv; ++k) {
        s[k] = (P.x[k] * dx + P.y[k] * dy) - half;
        any_out |= s[k] > 0.0;
    }
    if (!any_out) return true;
    int m = 0;
    for (int k = 0; k < P.nv; ++k) {
        const int kn = k + 1 == P.nv ? 0 : k + 1;
        const bool in_k = s[k] <= 0.0, in_n = s[kn] <= 0.0;
        if (m + 2 > BLD_MAXV) return false;
        if (in_k) {
            Q.x[m] = P.x[k];
            Q.y[m] = P.y[k];
            Q.g[m] = (!in_n && s[k] == 0.0) ? j : P.g[k];
            ++m;
            if (!in_n && s[k] < 0.0) {
                const double t = s[k] / (s[k] - s[kn]);
                Q.x[m] = P.x[k] + t * (P.x[kn] - P.x[k]);
                Q.y[m] = P.y[k] + t * (P.y[kn] - P.y[k]);
                Q.g[m] = j;
                ++m;
            }
        } else if (in_n && s[kn] < 0.0) {
            const double t = s[k] / (s[k] - s[kn]);
            Q.x[m] = P.x[k] + t * (P.x[kn] - P.x[k]);
            Q.y[m] = P.y[k] + t * (P.y[kn] - P.y[k]);
            Q.g[m] = P.g[k];
            ++m;
        }
    }
    Q.nv = m;
    for (int k = 0; k < m; ++k) {
        P.x[k] = Q.x[k];
        P.y[k] = Q.y[k];
        P.g[k] = Q.g[k];
    }
    P.nv = m;
    return true;
}

BD_HD double poly_rmax2(const Poly& P) {
    double r = 0.0;
    for (int k = 0; k < P.nv; ++k) {
        const double d = P.x[k] * P.x[k] + P.y[k] * P.y[k];
        r = d > r ? d : r;
    }
    return r;
}

// image shift of j as seen from i: pos[j] + s L is the image nearest pos[i]
BD_HD int64_t bld_shift(double pj, double pi, double L) { return -(int64_t)floor((pj - pi) / L + 0.5); }

template <class X>
BD_HD void bld_voronoi(X& x, BuildCtx& c, Poly& P, Poly& Q) {
    const BuildGeo& g = c.g;
    const int64_t n = g.n, ncx = g.ncx;
    // rings 0..ncx/2 visit every cell once (for even ncx the last ring's
    // offsets -r and +r are the same cell: -r is skipped)
    const int64_t max_ring = ncx / 2;
    for (int64_t i = x.tid(); i < n; i += x.nth()) {
        const double px = c.pos[2 * i], py = c.pos[2 * i + 1];
        const int64_t cx = bld_cell_coord(px, g), cy = bld_cell_coord(py, g);
        const double B = g.L;
        P.nv = 4;
        P.x[0] = -B; P.y[0] = -B; P.g[0] = -1;
        P.x[1] = B;  P.y[1] = -B; P.g[1] = -1;
        P.x[2] = B;  P.y[2] = B;  P.g[2] = -1;
        P.x[3] = -B; P.y[3] = B;  P.g[3] = -1;
        double rmax2 = poly_rmax2(P);
        bool done = false, bad = false;
        for (int64_t r = 0; r <= max_ring && !done && !bad; ++r) {
            for (int64_t oy = -r; oy <= r && !bad; ++oy) {
                const bool edge_row = oy == -r || oy == r;
                if (2 * r + 1 > ncx && oy == -r) continue;
                for (int64_t ox = -r; ox <= r && !bad; ox += edge_row ? 1 : 2 * (r > 0 ? r : 1)) {
                    if (2 * r + 1 > ncx && ox == -r) continue;
                    const int64_t qx = (cx + ox + ncx) % ncx, qy = (cy + oy + ncx) % ncx;
                    const int64_t q = qx + ncx * qy;
                    for (int32_t u = c.w.cell_start[q]; u < c.w.cell_start[q + 1]; ++u) {
                        const int64_t j = c.w.cell_pts[u];
                        if (j == i) continue;
                        const double dx = mi_ref(c.pos[2 * j] - px, g.L), dy = mi_ref(c.pos[2 * j + 1] - py, g.L);
                        const double d2 = dx * dx + dy * dy;
                        if (d2 == 0.0) {
                            bld_fail(x, c, i, BLD_COINCIDENT);
                            bad = true;
                            break;
                        }
                        if (d2 >= 4.0 * rmax2) continue;
                        if (!poly_clip(P, Q, dx, dy, 0.5 * d2, (int32_t)j)) {
                            bld_fail(x, c, i, BLD_POLY_OVERFLOW);
                            bad = true;
                            break;
                        }
                        rmax2 = poly_rmax2(P);
                    }
                }
            }
            // every unvisited point is >= r h away; it can only clip
            // vertices farther than r h / 2
            const double safe = (double)r * g.h;
            if (4.0 * rmax2 < safe * safe) done = true;
            // every cell visited: final if no second image of any point can
            // clip (second images are >= L/2 away), i.e. circumdiameters
            // < L/2 -- the reference audit's own bound (triangulation.py:470)
            if (r == max_ring && 16.0 * rmax2 < g.L * g.L) done = true;
        }
        if (bad) continue;
        if (!done) {
            bld_fail(x, c, i, BLD_TOO_SPARSE);
            continue;
        }
        // star: the cell's edges in CCW order, rotated to start at the
        // smallest neighbour
        if (P.nv > BLD_MAXD) {
            bld_fail(x, c, i, BLD_DEGREE_OVERFLOW);
            continue;
        }
        int k0 = 0;
        for (int k = 0; k < P.nv; ++k) {
            if (P.g[k] < 0) {
                bld_fail(x, c, i, BLD_TOO_SPARSE);
                bad = true;
                break;
            }
            if (P.g[k] < P.g[k0]) k0 = k;
        }
        if (bad) continue;
        int32_t* nb = c.w.nb + i * BLD_MAXD;
        int8_t* sh = c.w.sh + 2 * i * BLD_MAXD;
        for (int k = 0; k < P.nv; ++k) {
            const int64_t j = P.g[(k0 + k) % P.nv];
            const int64_t sx = bld_shift(c.pos[2 * j], px, g.L), sy = bld_shift(c.pos[2 * j + 1], py, g.L);
            if (sx < -1 || sx > 1 || sy < -1 || sy > 1) {
                bld_fail(x, c, i, BLD_SHIFT_RANGE);
                bad = true;
                break;
            }
            nb[k] = (int32_t)j;
            sh[2 * k] = (int8_t)sx;
            sh[2 * k + 1] = (int8_t)sy;
        }
        c.w.deg[i] = bad ? 0 : P.nv;
    }
    x.sync();
}

// ---- star queries ----------------------------------------------------------

struct StarRef {
    const int32_t* nb;
    const int8_t* sh;
    int d;
};

BD_HD StarRef star_of(const BuildCtx& c, int64_t v) {
    StarRef s;
    s.nb = c.w.nb + v * BLD_MAXD;
    s.sh = c.w.sh + 2 * v * BLD_MAXD;
    s.d = c.w.deg[v];
    return s;
}

// position of (u, shift sx, sy) in v's star, -1 if absent
BD_HD int star_find(const StarRef& s, int64_t u, int64_t sx, int64_t sy) {
    for (int k = 0; k < s.d; ++k)
        if (s.nb[k] == u && s.sh[2 * k] == sx && s.sh[2 * k + 1] == sy) return k;
    return -1;
}

// owned triangles / edges of v before star position p
BD_HD int owned_tris_before(const StarRef& s, int64_t v, int p) {
    int c = 0;
    for (int k = 0; k < p; ++k) {
        const int kn = k + 1 == s.d ? 0 : k + 1;
        c += (v < s.nb[k] && v < s.nb[kn]);
    }
    return c;
}

BD_HD int owned_edges_before(const StarRef& s, int64_t v, int p) {
    int c = 0;
    for (int k = 0; k < p; ++k) c += v < s.nb[k];
    return c;
}

// ---- phase 3: both-ends checks, owned counts --------------------------------

template <class X>
BD_HD void bld_check_count(X& x, BuildCtx& c) {
    const int64_t n = c.g.n;
    for (int64_t i = x.tid(); i < n; i += x.nth()) {
        const StarRef s = star_of(c, i);
        int32_t tc = 0, ec = 0;
        for (int m = 0; m < s.d; ++m) {
            const int mn = m + 1 == s.d ? 0 : m + 1;
            const int64_t a = s.nb[m], b = s.nb[mn];
            const int64_t sax = s.sh[2 * m], say = s.sh[2 * m + 1];
            const int64_t sbx = s.sh[2 * mn], sby = s.sh[2 * mn + 1];
            if (a == i || b == i || a == b || s.d < 3) {
                bld_fail(x, c, i, BLD_REPEATED_VERTEX);
                break;
            }
            // triangle (i, a, b) CCW is (a, b, i) in a's star: b precedes i
            const StarRef sa = star_of(c, a);
            const int p = star_find(sa, i, -sax, -say);
            if (p < 0) {
                bld_fail(x, c, i, BLD_ASYMMETRIC);
                break;
            }
            const int pp = p == 0 ? sa.d - 1 : p - 1;
            if (sa.nb[pp] != b || sa.sh[2 * pp] != sbx - sax || sa.sh[2 * pp + 1] != sby - say) {
                bld_fail(x, c, i, BLD_INCONSISTENT);
                break;
            }
            tc += (i < a && i < b);
            ec += i < a;
        }
        c.w.tcnt[i] = tc;
        c.w.ecnt[i] = ec;
    }
    x.sync();
}

// ---- phase 5: emit and link --------------------------------------------------

// id and slot layout of triangle (i, n_m, n_m+1) of i's star
struct TriRef {
    int64_t t;
    int rot;  // slot of i in the stored triangle (owner at slot 0)
};

BD_HD TriRef tri_ref(const BuildCtx& c, int64_t i, const StarRef& s, int m) {
    const int mn = m + 1 == s.d ? 0 : m + 1;
    const int64_t a = s.nb[m], b = s.nb[mn];
    TriRef r;
    if (i < a && i < b) {
        r.t = c.w.tcnt[i] + owned_tris_before(s, i, m);
        r.rot = 0;  // (i, a, b)
    } else if (a < b) {
        // owner a: stored (a, b, i); in a's star b sits at p with i at p+1
        const StarRef sa = star_of(c, a);
        const int p = star_find(sa, b, s.sh[2 * mn] - s.sh[2 * m], s.sh[2 * mn + 1] - s.sh[2 * m + 1]);
        r.t = c.w.tcnt[a] + owned_tris_before(sa, a, p);
        r.rot = 2;
    } else {
        // owner b: stored (b, i, a); in b's star i sits at p
        const StarRef sb = star_of(c, b);
        const int p = star_find(sb, i, -s.sh[2 * mn], -s.sh[2 * mn + 1]);
        r.t = c.w.tcnt[b] + owned_tris_before(sb, b, p);
        r.rot = 1;
    }
    return r;
}

// id of edge (i, n_m)
BD_HD int64_t edge_ref(const BuildCtx& c, int64_t i, const StarRef& s, int m) {
    const int64_t a = s.nb[m];
    if (i < a) return c.w.ecnt[i] + owned_edges_before(s, i, m);
    const StarRef sa = star_of(c, a);
    const int p = star_find(sa, i, -s.sh[2 * m], -s.sh[2 * m + 1]);
    return c.w.ecnt[a] + owned_edges_before(sa, a, p);
}

template <class X>
BD_HD void bld_emit(X& x, BuildCtx& c) {
    const int64_t n = c.g.n;
    const bd_tri_t& T = c.out;
    for (int64_t i = x.tid(); i < n; i += x.nth()) {
        const StarRef s = star_of(c, i);
        int64_t t = c.w.tcnt[i], e = c.w.ecnt[i];
        for (int m = 0; m < s.d; ++m) {
            const int mn = m + 1 == s.d ? 0 : m + 1, mp = m == 0 ? s.d - 1 : m - 1;
            const int64_t a = s.nb[m], b = s.nb[mn];
            if (i < a && i < b) {
                T.tri_v[3 * t] = (int32_t)i;
                T.tri_v[3 * t + 1] = (int32_t)a;
                T.tri_v[3 * t + 2] = (int32_t)b;
                T.tri_shift[6 * t] = 0;
                T.tri_shift[6 * t + 1] = 0;
                T.tri_shift[6 * t + 2] = s.sh[2 * m];
                T.tri_shift[6 * t + 3] = s.sh[2 * m + 1];
                T.tri_shift[6 * t + 4] = s.sh[2 * mn];
                T.tri_shift[6 * t + 5] = s.sh[2 * mn + 1];
                // edge opposite slot k: 0 -> (a, b), 1 -> (b, i), 2 -> (i, a)
                const StarRef sa = star_of(c, a);
                const int q = star_find(sa, b, s.sh[2 * mn] - s.sh[2 * m], s.sh[2 * mn + 1] - s.sh[2 * m + 1]);
                T.tri_edge[3 * t] = (int32_t)edge_ref(c, a, sa, q);
                T.tri_edge[3 * t + 1] = (int32_t)edge_ref(c, i, s, mn);
                T.tri_edge[3 * t + 2] = (int32_t)edge_ref(c, i, s, m);
                ++t;
            }
            if (i < a) {
                // side 0: (i, a, b) traverses i -> a; opposite vertex b
                // side 1: (i, n_m-1, a) traverses a -> i; opposite n_m-1
                const TriRef r0 = tri_ref(c, i, s, m), r1 = tri_ref(c, i, s, mp);
                T.edge_v[2 * e] = (int32_t)i;
                T.edge_v[2 * e + 1] = (int32_t)a;
                T.edge_tri[2 * e] = (int32_t)r0.t;
                T.edge_tri[2 * e + 1] = (int32_t)r1.t;
                // slot of the third vertex: i's slot + 2 in (i, a, b); i's slot + 1 in (i, c, a)
                T.edge_opp[2 * e] = (int8_t)((r0.rot + 2) % 3);
                T.edge_opp[2 * e + 1] = (int8_t)((r1.rot + 1) % 3);
                ++e;
            }
        }
    }
    x.sync();
}

// res = {status (0 / BD_ERR_BUILD), vertex, reason, 0}
template <class X>
BD_HD void tri_build(X& x, BuildCtx& c, Poly& P, Poly& Q, int64_t* res) {
    if (x.leader()) {
        c.w.ctl->status = 0;
        c.w.ctl->err_i = 0;
        c.w.ctl->err_k = 0;
    }
    x.sync();
    bld_bin(x, c);
    bld_voronoi(x, c, P, Q);
    if (x.ld(&c.w.ctl->status) == 0) {
        bld_check_count(x, c);
        if (x.ld(&c.w.ctl->status) == 0) {
            x.exclusive_scan(c.w.tcnt, c.g.n);
            x.exclusive_scan(c.w.ecnt, c.g.n);
            if (c.w.tcnt[c.g.n] != 2 * c.g.n || c.w.ecnt[c.g.n] != 3 * c.g.n || c.out.nt != 2 * c.g.n ||
                c.out.ne != 3 * c.g.n) {
                if (x.leader()) bld_fail(x, c, c.w.tcnt[c.g.n], BLD_EULER);
            } else {
                bld_emit(x, c);
            }
        }
    }
    x.sync();
    if (x.leader()) {
        res[0] = (int64_t)c.w.ctl->status;
        res[1] = (int64_t)c.w.ctl->err_i;
        res[2] = (int64_t)c.w.ctl->err_k;
        res[3] = 0;
    }
}

}  // namespace bd
