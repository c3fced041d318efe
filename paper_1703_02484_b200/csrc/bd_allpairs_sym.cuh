// bd_allpairs_sym.cuh -- FAST-SYM all-pairs force: Newton's third law on
// the shared factor r^-3, sorted slots, tile-uniform images.
//
// The force of _kernels.long_range_kernel (_kernels.py:26-59),
//     F_i = mu_i sum_{k != i} alpha_k r_ik / |r_ik|^3 ,
// is non-reciprocal (mu_i alpha_k != mu_k alpha_i) but its geometric factor
// w_ik = |r_ik|^-3 and the displacement r_ik = -r_ki are shared by the two
// directions of a pair.  Writing F_i = mu_i (A_i - B_i) with
//     A_i = sum over pairs where i is the receiver of  alpha_k w d ,
//     B_k = sum over pairs where k is the source   of  alpha_i w d ,
// every unordered pair is evaluated ONCE: 10 FP64 instructions for d, r^2
// and w (MUFU.RSQ64H + second-order correction), 3 for the receiver side
// and 3 for the source side -> 8 FP64 instructions per directed pair
// instead of the 12 of the directed FAST kernel (bd_allpairs_fast.cuh).
//
// Work decomposition (deterministic: every sum has a fixed order):
//  * slots are the Morton-sorted particles of the FAST path (same sort);
//    receiver blocks I of SY_BT = 512 slots, SY_R = 4 receivers per lane;
//  * block I pairs with blocks J = I + d (mod Mb), d = 1..D, D = Mb/2
//    (circulant: every unordered block pair exactly once; for even Mb the
//    d = D pairs belong to the lower block I < Mb/2), split into SY_S
//    chunks of d -> grid (Mb, SY_S); chunk 0 also does the diagonal block
//    J = I as directed pairs (receiver side only, k != i);
//  * the source tiles of J (SY_TS slots) stream through shared memory by
//    TMA; each lane owns SY_R receivers, so every source feeds SY_R pair
//    evaluations; the lane's source-side partial (summed over its
//    receivers) is reduced over the warp by a transposed shuffle tree, the
//    CTA adds its warps in warp order and writes one partial per
//    (d, source);
//  * k_sym_combine sums the SY_S receiver partials and the D source
//    partials of every slot in fixed order: F = mu (A - B).
// Multi-GPU: rank r of G owns the chunks [r S / G, (r+1) S / G) of every
// block (and with them a contiguous range of distances d); it writes the
// unscaled partial P_r = A_r - B_r of every slot, the ranks all-reduce P and
// finish F = mu P.  Deterministic for a given G; the sum order (and so the
// last bits) depends on G, unlike the directed FAST kernel.
#pragma once

#include "bd_allpairs_fast.cuh"

namespace bd {

struct alignas(16) SrcS {
    double x, y, a, mu;
};

struct alignas(16) SelS {  // receiver image selector (axis_select of both axes)
    double cx_le, cx_gt, cy_le, cy_gt;
    uint64_t Tx, Ty, amb;
    uint64_t tie;  // bit 0 / 1: some source lies within eps of the x / y breakpoint (k_tie_check)
};

// 4 receivers per lane in CTAs of 4 warps, 3 CTAs per SM (<= 170
// registers): 9.57 ms at cfg3 against 9.93 for 2 receivers in 8-warp CTAs at
// 2 per SM (each source read from shared memory feeds 4 pair evaluations and
// the source-side warp reduction is amortised over 32 pairs per lane)
#ifndef BD_SY_CT
#define BD_SY_CT 128
#endif
#ifndef BD_SY_R
#define BD_SY_R 4
#endif
constexpr int SY_R = BD_SY_R;          // receivers per lane
constexpr int SY_CT = BD_SY_CT;        // threads per CTA
constexpr int SY_BT = SY_CT * SY_R;    // receivers per block
#ifndef BD_SY_TS
#define BD_SY_TS 256
#endif
constexpr int SY_TS = BD_SY_TS;  // sources per shared-memory stage
#ifndef BD_SY_S
#define BD_SY_S 64
#endif
#ifndef BD_SY_MINB
#define BD_SY_MINB 3
#endif
constexpr int SY_S = BD_SY_S;  // chunks of the circulant distance range (grid.y)

BD_HD int64_t sym_blocks(int64_t n) { return (n + SY_BT - 1) / SY_BT; }
BD_HD int64_t sym_D(int64_t n) { return sym_blocks(n) / 2; }

// chunk and distance ranges of rank r of G (see the header comment)
struct SymRange {
    int c0, c1;      // chunks [c0, c1)
    int64_t d0, d1;  // source-side distances [d0, d1), d >= 1
};

BD_HD SymRange sym_range(int64_t n, int rank, int world);
BD_HD int64_t sym_tiles(int64_t n) { return (n + SY_TS - 1) / SY_TS; }
BD_HD int64_t sym_tie_buckets(int64_t n) { return n / 8 > 0 ? n / 8 : 1; }  // coordinate buckets per axis

struct SymWs {
    SortWs sort;     // cell sort of the FAST path (order, cells); its src/bbox/part3 are unused here
    SrcS* src;       // (n) sources in slot order
    SelS* sel;       // (n) receiver selectors in slot order
    uint64_t* bbox;  // (ntiles, 4) min/max bits of x and y per SY_TS tile
    double* tile_a;  // (ntiles) the tile's alpha when all its sources share it, else NaN
    int32_t* tcnt;   // (2 B + 1) coordinate buckets (x then y, B = sym_tie_buckets): counts -> offsets
    int32_t* tcur;   // (2 B) scatter cursors
    double* tval;    // (2 n) coordinates by bucket (x values, then y values)
    double* apart;   // (SY_S, n, 2) receiver-side partial sums per chunk
    double* bpart;   // (D, n, 2) source-side partial sums per circulant distance
    double* slot3;   // (n, 3) fx, fy, flag per slot
    double* part;    // (n, 2) P = A - B per slot (single GPU; ranks all-reduce their own)
};

BD_HD int64_t sym_ws_bytes(int64_t n) {
    const int64_t D = sym_D(n) > 0 ? sym_D(n) : 1;
    return fast_ws_bytes(n) + fs_align(32 * n) + fs_align(64 * n) + fs_align(32 * sym_tiles(n)) +
           fs_align(8 * sym_tiles(n)) + fs_align(4 * (2 * sym_tie_buckets(n) + 1)) +
           fs_align(8 * sym_tie_buckets(n)) + fs_align(16 * n) +
           fs_align(16 * n * SY_S) + fs_align(16 * n * D) + fs_align(24 * n) + fs_align(16 * n) + 256;
}

BD_HD SymWs sym_ws_carve(void* base, int64_t n) {
    SymWs w;
    w.sort = fast_ws_carve(base, n);
    char* b = (char*)(((uintptr_t)base + 255) & ~(uintptr_t)255) + fast_ws_bytes(n);
    const int64_t D = sym_D(n) > 0 ? sym_D(n) : 1;
    w.src = (SrcS*)b; b += fs_align(32 * n);
    w.sel = (SelS*)b; b += fs_align(64 * n);
    w.bbox = (uint64_t*)b; b += fs_align(32 * sym_tiles(n));
    w.tile_a = (double*)b; b += fs_align(8 * sym_tiles(n));
    w.tcnt = (int32_t*)b; b += fs_align(4 * (2 * sym_tie_buckets(n) + 1));
    w.tcur = (int32_t*)b; b += fs_align(8 * sym_tie_buckets(n));
    w.tval = (double*)b; b += fs_align(16 * n);
    w.apart = (double*)b; b += fs_align(16 * n * SY_S);
    w.bpart = (double*)b; b += fs_align(16 * n * D);
    w.slot3 = (double*)b; b += fs_align(24 * n);
    w.part = (double*)b;
    return w;
}

#if defined(__CUDACC__)

// one CTA per SY_TS tile of slots: sources, receiver selectors, tile box
__global__ void __launch_bounds__(SY_TS) k_sym_pack(const double* __restrict__ pos, const double* __restrict__ alpha,
                                                    const double* __restrict__ mu, int64_t n, double L, double lo,
                                                    double hi, SymWs w) {
    __shared__ uint64_t red[6][SY_TS / 32];
    const int64_t s = (int64_t)blockIdx.x * SY_TS + threadIdx.x;
    uint64_t xmin = ~0ull, xmax = 0, ymin = ~0ull, ymax = 0, amin = ~0ull, amax = 0;
    if (s < n) {
        const int64_t i = w.sort.order[s];
        const double x = pos[2 * i], y = pos[2 * i + 1];
        SrcS r;
        r.x = x;
        r.y = y;
        r.a = alpha[i];
        r.mu = mu[i];
        w.src[s] = r;
        const AxisSel sx = axis_select(x, L, lo, hi), sy = axis_select(y, L, lo, hi);
        SelS q;
        q.cx_le = x + sx.shift_le;
        q.cx_gt = x + sx.shift_gt;
        q.cy_le = y + sy.shift_le;
        q.cy_gt = y + sy.shift_gt;
        q.Tx = sx.T;
        q.Ty = sy.T;
        q.amb = (uint64_t)(sx.amb || sy.amb);
        q.tie = 0;
        w.sel[s] = q;
        xmin = xmax = dbits(x);
        ymin = ymax = dbits(y);
        amin = amax = dbits(r.a);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        xmin = min(xmin, __shfl_xor_sync(0xffffffffu, xmin, o));
        xmax = max(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
        ymin = min(ymin, __shfl_xor_sync(0xffffffffu, ymin, o));
        ymax = max(ymax, __shfl_xor_sync(0xffffffffu, ymax, o));
        amin = min(amin, __shfl_xor_sync(0xffffffffu, amin, o));
        amax = max(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        red[0][wid] = xmin;
        red[1][wid] = xmax;
        red[2][wid] = ymin;
        red[3][wid] = ymax;
        red[4][wid] = amin;
        red[5][wid] = amax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < SY_TS / 32; ++k) {
            xmin = min(xmin, red[0][k]);
            xmax = max(xmax, red[1][k]);
            ymin = min(ymin, red[2][k]);
            ymax = max(ymax, red[3][k]);
            amin = min(amin, red[4][k]);
            amax = max(amax, red[5][k]);
        }
        w.tile_a[blockIdx.x] = amin == amax ? bits_to_double(amin) : __longlong_as_double(0x7ff8000000000000ll);
        uint64_t* b = w.bbox + 4 * blockIdx.x;
        b[0] = xmin;
        b[1] = xmax;
        b[2] = ymin;
        b[3] = ymax;
    }
}

// ---- which receivers can meet an image tie ----------------------------------
// A pair is an image tie (source side's minimum image differs from the
// receiver side's) only if the source coordinate lies within eps of the
// receiver's breakpoint value (near_window).  Tiles whose box contains a
// breakpoint need the exact source-side arithmetic (EDGE mode) only when
// some source really is that close: one bucket pass over the coordinates
// (n buckets per axis over [0, L)) flags those receivers, per axis.  In
// lattice states many are flagged; once the particles have moved, none.

BD_HD double sym_tie_eps(double L) { return L * 0x1p-44; }

BD_DEV int64_t tie_bucket(double v, double L, int64_t B) {
    int64_t b = (int64_t)(v / L * (double)B);
    return b < 0 ? 0 : (b >= B ? B - 1 : b);
}

// x buckets [0, B), y buckets [B, 2B): one scan gives both offset tables
__global__ void k_tie_count(const double* __restrict__ pos, int64_t n, double L, SymWs w) {
    const int64_t B = sym_tie_buckets(n);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        atomicAdd(&w.tcnt[tie_bucket(pos[2 * i], L, B)], 1);
        atomicAdd(&w.tcnt[B + tie_bucket(pos[2 * i + 1], L, B)], 1);
    }
}

__global__ void k_tie_scatter(const double* __restrict__ pos, int64_t n, double L, SymWs w) {
    const int64_t B = sym_tie_buckets(n);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = pos[2 * i], y = pos[2 * i + 1];
        const int64_t bx = tie_bucket(x, L, B), by = B + tie_bucket(y, L, B);
        w.tval[w.tcnt[bx] + atomicAdd(&w.tcur[bx], 1)] = x;
        w.tval[w.tcnt[by] + atomicAdd(&w.tcur[by], 1)] = y;
    }
}

BD_DEV bool tie_axis(const SymWs& w, int64_t n, double L, uint64_t T, int axis) {
    if (T == ~0ull) return false;
    const int64_t B = sym_tie_buckets(n);
    const double tv = bits_to_double(T), eps = sym_tie_eps(L);
    const double lo_v = tv - eps > 0.0 ? tv - eps : 0.0, hi_v = tv + eps;
    const uint64_t lo = dbits(lo_v), hi = dbits(hi_v);
    const int32_t* off = w.tcnt + axis * B;
    const double* val = w.tval;
    for (int64_t b = tie_bucket(lo_v, L, B); b <= tie_bucket(hi_v, L, B); ++b)
        for (int32_t k = off[b]; k < off[b + 1]; ++k) {
            const uint64_t v = dbits(val[k]);
            if (v >= lo && v <= hi) return true;
        }
    return false;
}

__global__ void k_tie_check(int64_t n, double L, SymWs w) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const SelS q = w.sel[s];
        w.sel[s].tie = (uint64_t)tie_axis(w, n, L, q.Tx, 0) | ((uint64_t)tie_axis(w, n, L, q.Ty, 1) << 1);
    }
}

// r^-3 from r^2: y0 = MUFU.RSQ64H (~2^-22), e = 1 - r2 y0^2,
// r^-3 = y0^3 (1 + 1.5 e + 1.875 e^2) (+ O(e^3) ~ 1e-19)
BD_DEV double inv_r3(double r2) {
    const double y0 = rsqrt_mufu(r2);
    const double t = y0 * y0;
    const double e = fma(-r2, t, 1.0);
    const double y3 = t * y0;
    return y3 * fma(fma(1.875, e, 1.5), e, 1.0);
}

// SY_R receivers per lane (slots lane + 32 m of the warp's 32 SY_R): every
// source read from shared memory feeds SY_R pair evaluations, and the
// source-side partial of a lane is the sum over its receivers before the
// warp reduction (so the reduction is amortised over 32 SY_R pairs).
struct SymRecv {
    double cx_le[SY_R], cx_gt[SY_R], cy_le[SY_R], cy_gt[SY_R];
    uint64_t Tx[SY_R], Ty[SY_R];
    uint32_t tie[SY_R];  // SelS.tie
    double a[SY_R];   // alpha of the receiver (source-side factor); 0 for an inactive slot
    double ax[SY_R], ay[SY_R];  // receiver-side accumulators A
    double sx[SY_R], sy[SY_R];  // factored tiles: sum of w d over the tile (A += alpha_tile s)
};

enum { SY_UNIFORM = 0, SY_SELECT = 1, SY_EDGE_M = 2, SY_GENERIC = 3 };

// raw receiver coordinate from its selector: one of the two shifted copies is unshifted
BD_DEV double raw_coord(double c_le, double c_gt, double L) { return c_gt < L ? c_gt : c_le; }

// One source against the lane's receivers.  Receiver side: A += alpha_k w d.
// Source side: returns sum_m alpha_m w d_src (x, y) for the warp reduction.
// d_src is minus the source's OWN minimum-image displacement to the
// receiver; it equals d except at image ties (fl(d / L) within ulps of
// +-1/2, e.g. lattice pairs exactly L/2 apart), where the reference's two
// directions do not use mirror images.  Such pairs have the source within
// ~ulps(L) of the receiver's breakpoint value, so per (warp, tile):
//   UNIFORM -- no breakpoint inside or near the tile's box: one image shift
//              per receiver, d_src = d;
//   SELECT  -- a breakpoint inside the box, none near a source: per-pair
//              image from the breakpoints (integer compares), d_src = d;
//   EDGE    -- a breakpoint within eps of the box: per-pair image and d_src
//              from the exact min-image arithmetic of the source side;
//   GENERIC -- exact min-image arithmetic on both sides (receivers within
//              ulps of L/2 have ambiguous breakpoints; essentially never).

// FACT: the tile's sources share one alpha and the warp's receivers share
// one alpha, so both factors leave the pair loop: the receiver side sums
// w d per tile (scaled by the tile's alpha at its end), the source side sums
// w d_src over the warp (scaled by the warp's alpha after the reduction).
// 14 FP64 instructions per unordered pair instead of 16.
template <int MODE, bool FACT = false>
BD_DEV void sym_pair(SymRecv& r, const SrcS& s, const double* cx, const double* cy, const double* Ll, double& bx,
                     double& by) {
    double dx[SY_R], dy[SY_R];
#pragma unroll
    for (int m = 0; m < SY_R; ++m) {
        if (MODE == SY_UNIFORM) {
            dx[m] = cx[m] - s.x;
            dy[m] = cy[m] - s.y;
        } else if (MODE == SY_GENERIC) {
            dx[m] = mi_fast(raw_coord(r.cx_le[m], r.cx_gt[m], Ll[0]) - s.x, Ll[0], Ll[1], Ll[2]);
            dy[m] = mi_fast(raw_coord(r.cy_le[m], r.cy_gt[m], Ll[0]) - s.y, Ll[0], Ll[1], Ll[2]);
        } else {
            dx[m] = (dbits(s.x) <= r.Tx[m] ? r.cx_le[m] : r.cx_gt[m]) - s.x;
            dy[m] = (dbits(s.y) <= r.Ty[m] ? r.cy_le[m] : r.cy_gt[m]) - s.y;
        }
    }
    bx = 0.0;
    by = 0.0;
#pragma unroll
    for (int m = 0; m < SY_R; ++m) {
        double sxm = dx[m], sym = dy[m];
        if (MODE == SY_EDGE_M || MODE == SY_GENERIC) {  // the source side's own exact image
            sxm = -mi_fast(s.x - raw_coord(r.cx_le[m], r.cx_gt[m], Ll[0]), Ll[0], Ll[1], Ll[2]);
            sym = -mi_fast(s.y - raw_coord(r.cy_le[m], r.cy_gt[m], Ll[0]), Ll[0], Ll[1], Ll[2]);
        }
        const double w = inv_r3(fma(dx[m], dx[m], dy[m] * dy[m]));
        if (FACT) {
            r.sx[m] = fma(w, dx[m], r.sx[m]);
            r.sy[m] = fma(w, dy[m], r.sy[m]);
            bx = fma(w, sxm, bx);
            by = fma(w, sym, by);
        } else {
            const double ta = s.a * w;
            r.ax[m] = fma(ta, dx[m], r.ax[m]);
            r.ay[m] = fma(ta, dy[m], r.ay[m]);
            const double tb = r.a[m] * w;
            bx = fma(tb, sxm, bx);
            by = fma(tb, sym, by);
        }
    }
}

// Does [b0, b1] (source coordinate bits) come within eps (absolute) of the
// breakpoint T?  Image ties need |fl(x_i - s)| within ulps(L) of L/2, i.e. s
// within ~ulps(L) of the breakpoint VALUE (a bit-pattern distance would be
// wrong for small s).  T = ~0: no breakpoint, no tie.
BD_DEV bool near_window(uint64_t b0, uint64_t b1, uint64_t T, double eps) {
    if (T == ~0ull) return false;
    const double tv = bits_to_double(T);
    const uint64_t lo = dbits(tv - eps > 0.0 ? tv - eps : 0.0), hi = dbits(tv + eps);
    return !(b1 < lo || b0 > hi);
}

// diagonal block (J == I): directed, receiver side only, k != i
template <int MODE>
BD_DEV void sym_diag(SymRecv& r, const SrcS& s, int64_t k, const int64_t* slot, const double* cx,
                     const double* cy, const double* Ll) {
#pragma unroll
    for (int m = 0; m < SY_R; ++m) {
        double dx, dy;
        if (MODE == SY_GENERIC) {
            dx = mi_fast(raw_coord(r.cx_le[m], r.cx_gt[m], Ll[0]) - s.x, Ll[0], Ll[1], Ll[2]);
            dy = mi_fast(raw_coord(r.cy_le[m], r.cy_gt[m], Ll[0]) - s.y, Ll[0], Ll[1], Ll[2]);
        } else {
            dx = (dbits(s.x) <= r.Tx[m] ? r.cx_le[m] : r.cx_gt[m]) - s.x;
            dy = (dbits(s.y) <= r.Ty[m] ? r.cy_le[m] : r.cy_gt[m]) - s.y;
        }
        double ta = s.a * inv_r3(fma(dx, dx, dy * dy));
        ta = k == slot[m] ? 0.0 : ta;
        r.ax[m] = fma(ta, dx, r.ax[m]);
        r.ay[m] = fma(ta, dy, r.ay[m]);
    }
}

// Transposed warp reduction of 8 per-lane values, one per source, without
// selects: lane l holds in v[u] the partial of source u ^ g(l),
// g(l) = (l >> 2) & 7 (the pair loop visits the sources in that order), so
// each halving step exchanges a fixed register half.  After it, lane l holds
// the warp sum for source g(l).  9 shuffles + 9 adds for 8 sums (a
// butterfly per value: 40 + 40).
BD_DEV double tree8(const double v[8]) {
    double h[4], q[2];
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = v[j] + __shfl_xor_sync(0xffffffffu, v[j + 4], 16);
#pragma unroll
    for (int j = 0; j < 2; ++j) q[j] = h[j] + __shfl_xor_sync(0xffffffffu, h[j + 2], 8);
    double r = q[0] + __shfl_xor_sync(0xffffffffu, q[1], 4);
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    return r;
}

BD_DEV double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr int SY_G = 8;  // sources per transposed reduction

// a tile of `cnt` sources: pair evaluations + warp sums of the source side into bws[2*j .. 2*j+1]
// (FACT: ta = the tile's alpha, wa = the warp's receiver alpha)
template <int MODE, bool FACT = false>
BD_DEV void sym_tile(SymRecv& r, const SrcS* sm, int cnt, const double* cx, const double* cy, const double* Ll,
                     double* bws, int lane, double ta = 0.0, double wa = 0.0) {
    int j = 0;
    const int g = (lane >> 2) & 7;  // this lane visits source j + (u ^ g) at step u
    if (FACT) {
#pragma unroll
        for (int m = 0; m < SY_R; ++m) {
            r.sx[m] = 0.0;
            r.sy[m] = 0.0;
        }
    }
    for (; j + SY_G <= cnt; j += SY_G) {
        double bx[SY_G], by[SY_G];
#pragma unroll
        for (int u = 0; u < SY_G; ++u) sym_pair<MODE, FACT>(r, sm[j + (u ^ g)], cx, cy, Ll, bx[u], by[u]);
        double sx = tree8(bx), sy = tree8(by);
        if (FACT) {
            sx *= wa;
            sy *= wa;
        }
        if ((lane & 3) == 0) {
            const int k = j + g;
            bws[2 * k] = sx;
            bws[2 * k + 1] = sy;
        }
    }
    for (; j < cnt; ++j) {
        double bx, by;
        sym_pair<MODE, FACT>(r, sm[j], cx, cy, Ll, bx, by);
        double sx = warp_sum(bx), sy = warp_sum(by);
        if (FACT) {
            sx *= wa;
            sy *= wa;
        }
        if (lane == 0) {
            bws[2 * j] = sx;
            bws[2 * j + 1] = sy;
        }
    }
    if (FACT) {
#pragma unroll
        for (int m = 0; m < SY_R; ++m) {
            r.ax[m] = fma(ta, r.sx[m], r.ax[m]);
            r.ay[m] = fma(ta, r.sy[m], r.ay[m]);
        }
    }
}

BD_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// TMA of source tile t (SY_TS slots; fewer or none past n) into stage st
BD_DEV void sym_issue(const SymWs& w, int64_t n, int64_t t, SrcS* tiles, uint64_t* bars, int st) {
    const int64_t cnt = (t + 1) * SY_TS <= n ? SY_TS : (t * SY_TS < n ? n - t * SY_TS : 0);
    mbar_expect_tx(&bars[st], (uint32_t)(cnt * sizeof(SrcS)));
    if (cnt) bulk_g2s(tiles + st * SY_TS, w.src + t * SY_TS, (uint32_t)(cnt * sizeof(SrcS)), &bars[st]);
}

constexpr int SY_NW2 = SY_CT / 32;   // warps per CTA
// dynamic smem: 2 source stages + 2 buffers of per-warp source-side sums
#ifndef BD_SY_NB
#define BD_SY_NB 2
#endif
constexpr int SY_NB = BD_SY_NB;  // source-sum buffers (1: one more CTA barrier per tile, half the smem)
constexpr int SY_SMEM = 2 * SY_TS * (int)sizeof(SrcS) + SY_NB * SY_NW2 * SY_TS * 16;

// grid (Mb, SY_S), SY_CT threads; warp v of block I owns slots I*SY_BT + 64 v + {lane, lane + 32}
__global__ void __launch_bounds__(SY_CT, BD_SY_MINB) k_allpairs_sym(SymWs w, int64_t n, double L, double lo, double hi,
                                                                     int chunk0) {
    extern __shared__ __align__(128) unsigned char sy_smem[];
    SrcS* tiles = reinterpret_cast<SrcS*>(sy_smem);                              // [2][SY_TS]
    double* bw = reinterpret_cast<double*>(sy_smem + 2 * SY_TS * sizeof(SrcS));  // [2][SY_NW2][SY_TS][2]
    __shared__ __align__(8) uint64_t bars[2];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t Mb = sym_blocks(n), D = sym_D(n);
    const int64_t I = blockIdx.x;
    const int chunk = chunk0 + (int)blockIdx.y;

    SymRecv r;
    int64_t slot[SY_R];
    bool act[SY_R], amb = false;
#pragma unroll
    for (int m = 0; m < SY_R; ++m) {
        slot[m] = I * SY_BT + 32 * SY_R * wid + lane + 32 * m;
        act[m] = slot[m] < n;
        const int64_t sl = act[m] ? slot[m] : I * SY_BT;
        const SelS q = w.sel[sl];
        r.cx_le[m] = q.cx_le;
        r.cx_gt[m] = q.cx_gt;
        r.cy_le[m] = q.cy_le;
        r.cy_gt[m] = q.cy_gt;
        r.Tx[m] = q.Tx;
        r.Ty[m] = q.Ty;
        r.tie[m] = (uint32_t)q.tie;
        r.a[m] = act[m] ? w.src[sl].a : 0.0;
        r.ax[m] = 0.0;
        r.ay[m] = 0.0;
        amb |= act[m] && q.amb;
    }
    const double Ll[3] = {L, lo, hi};
    // the warp's receivers all active with one alpha: factored tiles possible
    const double wa = __shfl_sync(0xffffffffu, r.a[0], 0);
    bool wone = true;
#pragma unroll
    for (int m = 0; m < SY_R; ++m) wone &= act[m] && r.a[m] == wa;
    const bool wfact = __all_sync(0xffffffffu, wone);

    // this chunk's distances [d0, d1); chunk 0 adds the diagonal block (d = 0)
    const int64_t per = (D + SY_S - 1) / SY_S;
    const int64_t d0 = chunk == 0 ? 0 : 1 + (int64_t)chunk * per;
    const int64_t d1 = 1 + ((int64_t)chunk + 1) * per < D + 1 ? 1 + ((int64_t)chunk + 1) * per : D + 1;
    const bool even = (Mb & 1) == 0;
    constexpr int64_t tpb = SY_BT / SY_TS;  // source tiles per block
    const int64_t nq = d1 > d0 ? (d1 - d0) * tpb : 0;

    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const bool wamb = __any_sync(0xffffffffu, amb);
    if (threadIdx.x == 0)
        for (int64_t qi = 0; qi < 2 && qi < nq; ++qi)
            sym_issue(w, n, ((I + d0 + qi / tpb) % Mb) * tpb + qi % tpb, tiles, bars, (int)qi);

    for (int64_t qi = 0; qi < nq; ++qi) {
        const int st = (int)(qi & 1);
        const int64_t d = d0 + qi / tpb;
        const int64_t J = (I + d) % Mb;
        const int64_t t = J * tpb + qi % tpb;
        const int64_t base = t * SY_TS;
        const int cnt = (int)((t + 1) * SY_TS <= n ? SY_TS : (base < n ? n - base : 0));
        const bool use = !(even && d == D && d > 0 && I >= Mb / 2) && cnt > 0;
        const uint64_t* bb = w.bbox + 4 * t;
        const uint64_t bx0 = bb[0], bx1 = bb[1], by0 = bb[2], by1 = bb[3];
        const double ta = w.tile_a[t];
        const bool fact = wfact && ta == ta;  // NaN: mixed tile
        mbar_wait(&bars[st], (uint32_t)((qi >> 1) & 1));
        const SrcS* sm = tiles + st * SY_TS;
        const int sb = SY_NB == 1 ? 0 : st;
        double* bws = bw + ((size_t)sb * SY_NW2 + wid) * SY_TS * 2;
        if (use) {
            double cx[SY_R], cy[SY_R];
            bool uni = true, edge = false;
            const double eps = sym_tie_eps(L);  // >> the ulps of L in which image ties live
#pragma unroll
            for (int m = 0; m < SY_R; ++m) {
                const bool xle = bx1 <= r.Tx[m], xgt = bx0 > r.Tx[m], yle = by1 <= r.Ty[m], ygt = by0 > r.Ty[m];
                uni &= (xle || xgt) && (yle || ygt);
                edge |= ((r.tie[m] & 1) && near_window(bx0, bx1, r.Tx[m], eps)) ||
                        ((r.tie[m] & 2) && near_window(by0, by1, r.Ty[m], eps));
                cx[m] = xle ? r.cx_le[m] : r.cx_gt[m];
                cy[m] = yle ? r.cy_le[m] : r.cy_gt[m];
            }
            const bool any_edge = __any_sync(0xffffffffu, edge);
            const bool all_uni = __all_sync(0xffffffffu, uni);
            if (d == 0) {
                if (wamb) {
                    for (int j = 0; j < cnt; ++j) sym_diag<SY_GENERIC>(r, sm[j], base + j, slot, cx, cy, Ll);
                } else {
                    for (int j = 0; j < cnt; ++j) sym_diag<SY_SELECT>(r, sm[j], base + j, slot, cx, cy, Ll);
                }
            } else if (wamb) {
                sym_tile<SY_GENERIC>(r, sm, cnt, cx, cy, Ll, bws, lane);
            } else if (any_edge) {
                sym_tile<SY_EDGE_M>(r, sm, cnt, cx, cy, Ll, bws, lane);
            } else if (all_uni) {
                if (fact)
                    sym_tile<SY_UNIFORM, true>(r, sm, cnt, cx, cy, Ll, bws, lane, ta, wa);
                else
                    sym_tile<SY_UNIFORM>(r, sm, cnt, cx, cy, Ll, bws, lane);
            } else {
                if (fact)
                    sym_tile<SY_SELECT, true>(r, sm, cnt, cx, cy, Ll, bws, lane, ta, wa);
                else
                    sym_tile<SY_SELECT>(r, sm, cnt, cx, cy, Ll, bws, lane);
            }
        }
        __syncthreads();  // stage st consumed; the warps' source-side sums of tile qi complete
        if (threadIdx.x == 0 && qi + 2 < nq) {
            fence_proxy_async_smem();
            sym_issue(w, n, ((I + d0 + (qi + 2) / tpb) % Mb) * tpb + (qi + 2) % tpb, tiles, bars, st);
        }
        if (use && d > 0) {
            // CTA sum of the warp sums (warp order) -> one partial per (d, source)
            const double* bt = bw + (size_t)sb * SY_NW2 * SY_TS * 2;
            for (int e = threadIdx.x; e < 2 * cnt; e += SY_CT) {
                double v = 0.0;
#pragma unroll
                for (int ww = 0; ww < SY_NW2; ++ww) v += bt[(size_t)ww * SY_TS * 2 + e];
                w.bpart[(size_t)(d - 1) * n * 2 + (size_t)base * 2 + e] = v;
            }
        }
        // this stage's sum buffer is written again two tiles later, after the next __syncthreads
        if (SY_NB == 1) __syncthreads();
    }
#pragma unroll
    for (int m = 0; m < SY_R; ++m) {
        if (!act[m]) continue;
        w.apart[(size_t)chunk * n * 2 + 2 * slot[m]] = r.ax[m];
        w.apart[(size_t)chunk * n * 2 + 2 * slot[m] + 1] = r.ay[m];
    }
}

// P = A - B per slot over this rank's chunks / distances, fixed order -> part (n, 2)
__global__ void k_sym_partial(int64_t n, SymWs w, SymRange g, double* __restrict__ part) {
    const int64_t Mb = sym_blocks(n), D = sym_D(n);
    const bool even = (Mb & 1) == 0;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        // 16-byte loads, 8 in flight (the sums keep their sequential order)
        double ax = 0.0, ay = 0.0, bx = 0.0, by = 0.0;
        const double2* ap = reinterpret_cast<const double2*>(w.apart) + s;
#pragma unroll 8
        for (int c = g.c0; c < g.c1; ++c) {
            const double2 v = __ldcs(ap + (size_t)c * n);
            ax += v.x;
            ay += v.y;
        }
        const int64_t J = s / SY_BT;
        // d = D of an even block count belongs to the lower block only
        const int64_t dend = (even && g.d1 == D + 1 && (J - D + Mb) % Mb >= Mb / 2) ? D : g.d1;
        const double2* bp = reinterpret_cast<const double2*>(w.bpart) + s;
#pragma unroll 8
        for (int64_t d = g.d0; d < dend; ++d) {
            const double2 v = __ldcs(bp + (size_t)(d - 1) * n);
            bx += v.x;
            by += v.y;
        }
        part[2 * s] = ax - bx;
        part[2 * s + 1] = ay - by;
    }
}

// F = mu P per slot -> slot3 (fx, fy, flag)
__global__ void k_sym_finish(int64_t n, SymWs w, const double* __restrict__ part) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const double mu = w.src[s].mu;
        const double fx = mu * part[2 * s], fy = mu * part[2 * s + 1];
        w.slot3[3 * s] = fx;
        w.slot3[3 * s + 1] = fy;
        w.slot3[3 * s + 2] = (isfinite(fx) && isfinite(fy)) ? 0.0 : -1.0;
    }
}

#endif  // __CUDACC__

BD_HD SymRange sym_range(int64_t n, int rank, int world) {
    SymRange g;
    g.c0 = (int)((int64_t)rank * SY_S / world);
    g.c1 = (int)((int64_t)(rank + 1) * SY_S / world);
    const int64_t D = sym_D(n), per = (D + SY_S - 1) / SY_S;
    const int64_t a = g.c0 == 0 ? 1 : 1 + (int64_t)g.c0 * per;  // chunk c >= 1 starts at 1 + c per
    const int64_t b = 1 + (int64_t)g.c1 * per;
    g.d0 = a < D + 1 ? a : D + 1;
    g.d1 = b < D + 1 ? b : D + 1;
    if (g.c1 <= g.c0) g.d1 = g.d0;
    return g;
}

}  // namespace bd
