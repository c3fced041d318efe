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
//  * slots are the particles sorted by (alpha group, Morton cell); receiver
//    blocks I of SY_BT = 512 slots, SY_R = 4 receivers per lane;
//  * block I pairs with blocks J = I + d (mod Mb), d = 1..D, D = Mb/2
//    (circulant: every unordered block pair exactly once; for even Mb the
//    d = D pairs belong to the lower block I < Mb/2), split into SY_S
//    chunks of d -> grid (Mb, SY_S); the diagonal blocks J = I (directed
//    pairs, receiver side only, k != i) are a separate set of Mb CTAs
//    (chunk index SY_S), so they can be spread over ranks like the rest;
//  * the source tiles of J (SY_TS slots) stream through shared memory by
//    TMA; each lane owns SY_R receivers, so every source feeds SY_R pair
//    evaluations; the lane's source-side partial (summed over its
//    receivers) is reduced over the warp by a transposed shuffle tree, the
//    CTA adds its warps in warp order and writes one partial per
//    (d, source);
//  * k_sym_partial sums the receiver partials (chunks, then the diagonal)
//    and the source partials (ascending d) of every slot in fixed order:
//    P = A - B; k_sym_finish: F = mu P.
// Registers: only the per-tile image of each receiver (UNIFORM) or its
// selector (per-pair modes, in passes of fewer receivers) is live in the
// pair loop; the lanes' running receiver sums live in shared memory.
// <= 128 registers -> 4 CTAs of 4 warps per SM (16 warps).
// Multi-GPU: rank r of G owns the chunks [r S / G, (r+1) S / G) (S = the
// chunks in use, min(SY_S, D)) of every
// block and the diagonal blocks [r Mb / G, (r+1) Mb / G); it writes the
// unscaled partial P_r = A_r - B_r of every slot, the ranks all-reduce P and
// finish F = mu P.  Deterministic for a given G; the sum order (and so the
// last bits) depends on G, unlike the directed FAST kernel.
#pragma once

#include "bd_allpairs_fast.cuh"

namespace bd {

struct alignas(16) SymXY {  // a position (16-byte loads)
    double x, y;
};

struct SrcS {  // one source as the pair loop sees it (shared-memory stage: xy and alpha arrays)
    double x, y, a;
};

struct alignas(16) SelS {  // receiver image selector (axis_select of both axes)
    double cx_le, cx_gt, cy_le, cy_gt;
    uint64_t Tx, Ty, amb;
    uint64_t tie;  // bit 0 / 1: some source lies within eps of the x / y breakpoint (k_sym_pack)
};

// 4 receivers per lane in CTAs of 4 warps (each source read from shared
// memory feeds 4 pair evaluations and the source-side warp reduction is
// amortised over 32 pairs per lane), 4 CTAs per SM
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
// sources per image-mode decision (a sub-tile of a stage with its own bounding
// box): smaller boxes straddle fewer receiver breakpoints, so less of the work
// runs the per-pair image modes
#ifndef BD_SY_SUB
#define BD_SY_SUB 256
#endif
constexpr int SY_SUB = BD_SY_SUB;
static_assert(SY_TS % SY_SUB == 0 && SY_SUB % 32 == 0, "sub-tiles of whole warps");
#ifndef BD_SY_S
#define BD_SY_S 64
#endif
#ifndef BD_SY_MINB
#define BD_SY_MINB 4
#endif
constexpr int SY_S = BD_SY_S;  // chunks of the circulant distance range (grid.y)

BD_HD int64_t sym_blocks(int64_t n) { return (n + SY_BT - 1) / SY_BT; }
BD_HD int64_t sym_D(int64_t n) { return sym_blocks(n) / 2; }
// chunks of the distance range actually used (<= SY_S, none empty) and distances per chunk
BD_HD int64_t sym_chunks(int64_t n) { return sym_D(n) < SY_S ? (sym_D(n) > 0 ? sym_D(n) : 1) : SY_S; }
BD_HD int64_t sym_per(int64_t n) { return (sym_D(n) + sym_chunks(n) - 1) / sym_chunks(n); }

// chunk and distance ranges of rank r of G (see the header comment)
struct SymRange {
    int c0, cs, nch;  // chunks c0, c0 + cs, c0 + 2 cs, ... (nch of them; interleaved over the ranks)
    int64_t i0, i1;   // diagonal blocks [i0, i1)
};

BD_HD SymRange sym_range(int64_t n, int rank, int world);
BD_HD int64_t sym_tiles(int64_t n) { return (n + SY_TS - 1) / SY_TS; }
BD_HD int64_t sym_subs(int64_t n) { return sym_tiles(n) * (SY_TS / SY_SUB); }
BD_HD int64_t sym_tie_buckets(int64_t n) { return n / 8 > 0 ? n / 8 : 1; }  // coordinate buckets per axis

struct SymWs {
    SortWs sort;     // cell sort of the FAST path (order, cells); its src/bbox/part3 are unused here
    SymXY* sxy;    // (n) source positions in slot order
    double* sa;      // (n) source alpha in slot order
    double* smu;     // (n) mu in slot order
    SelS* sel;       // (n) receiver selectors in slot order
    uint64_t* bbox;  // (nsubs, 4) min/max bits of x and y per SY_SUB sub-tile
    double* tile_a;  // (ntiles) the tile's alpha when all its sources share it, else NaN
    int32_t* tcnt;   // (2 B + 1) coordinate buckets (x then y, B = sym_tie_buckets): counts -> offsets
    int32_t* tcur;   // (2 B) scatter cursors
    double* tval;    // (2 n) coordinates by bucket (x values, then y values)
    double* apart;   // (SY_S + 1, n, 2) receiver-side partial sums per chunk (+ the diagonal block)
    double* bpart;   // (D, n, 2) source-side partial sums per circulant distance
    double* part;    // (n, 2) P = A - B per slot (single GPU; ranks all-reduce their own)
};

BD_HD int64_t sym_ws_bytes(int64_t n) {
    const int64_t D = sym_D(n) > 0 ? sym_D(n) : 1;
    return fast_ws_bytes(n) + fs_align(16 * n) + 2 * fs_align(8 * n) + fs_align(64 * n) + fs_align(32 * sym_subs(n)) +
           fs_align(8 * sym_tiles(n)) + fs_align(4 * (2 * sym_tie_buckets(n) + 1)) +
           fs_align(8 * sym_tie_buckets(n)) + fs_align(16 * n) +
           fs_align(16 * n * (SY_S + 1)) + fs_align(16 * n * D) + fs_align(16 * n) + 256;
}

BD_HD SymWs sym_ws_carve(void* base, int64_t n) {
    SymWs w;
    w.sort = fast_ws_carve(base, n);
    char* b = (char*)(((uintptr_t)base + 255) & ~(uintptr_t)255) + fast_ws_bytes(n);
    const int64_t D = sym_D(n) > 0 ? sym_D(n) : 1;
    w.sxy = (SymXY*)b; b += fs_align(16 * n);
    w.sa = (double*)b; b += fs_align(8 * n);
    w.smu = (double*)b; b += fs_align(8 * n);
    w.sel = (SelS*)b; b += fs_align(64 * n);
    w.bbox = (uint64_t*)b; b += fs_align(32 * sym_subs(n));
    w.tile_a = (double*)b; b += fs_align(8 * sym_tiles(n));
    w.tcnt = (int32_t*)b; b += fs_align(4 * (2 * sym_tie_buckets(n) + 1));
    w.tcur = (int32_t*)b; b += fs_align(8 * sym_tie_buckets(n));
    w.tval = (double*)b; b += fs_align(16 * n);
    w.apart = (double*)b; b += fs_align(16 * n * (SY_S + 1));
    w.bpart = (double*)b; b += fs_align(16 * n * D);
    w.part = (double*)b;
    return w;
}

#if defined(__CUDACC__)

BD_DEV bool tie_axis(const SymWs& w, int64_t n, double L, uint64_t T, int axis);

// one CTA per SY_TS tile of slots: sources, receiver selectors (with their
// tie bits: the coordinate buckets are filled by k_sym_scatter), tile box
__global__ void __launch_bounds__(SY_TS) k_sym_pack(const double* __restrict__ pos, const double* __restrict__ alpha,
                                                    const double* __restrict__ mu, int64_t n, double L, double lo,
                                                    double hi, SymWs w) {
    __shared__ uint64_t red[6][SY_TS / 32];
    const int64_t s = (int64_t)blockIdx.x * SY_TS + threadIdx.x;
    uint64_t xmin = ~0ull, xmax = 0, ymin = ~0ull, ymax = 0, amin = ~0ull, amax = 0;
    if (s < n) {
        const int64_t i = w.sort.order[s];
        const double x = pos[2 * i], y = pos[2 * i + 1];
        const double a = alpha[i];
        w.sxy[s] = SymXY{x, y};
        w.sa[s] = a;
        w.smu[s] = mu[i];
        const AxisSel sx = axis_select(x, L, lo, hi), sy = axis_select(y, L, lo, hi);
        SelS q;
        q.cx_le = x + sx.shift_le;
        q.cx_gt = x + sx.shift_gt;
        q.cy_le = y + sy.shift_le;
        q.cy_gt = y + sy.shift_gt;
        q.Tx = sx.T;
        q.Ty = sy.T;
        q.amb = (uint64_t)(sx.amb || sy.amb);
        q.tie = (uint64_t)tie_axis(w, n, L, q.Tx, 0) | ((uint64_t)tie_axis(w, n, L, q.Ty, 1) << 1);
        w.sel[s] = q;
        xmin = xmax = dbits(x);
        ymin = ymax = dbits(y);
        amin = amax = dbits(a);
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
    constexpr int WPS = SY_SUB / 32;  // warps per sub-tile
    if (threadIdx.x < SY_TS / SY_SUB) {
        const int k0 = threadIdx.x * WPS;
        uint64_t sx0 = red[0][k0], sx1 = red[1][k0], sy0 = red[2][k0], sy1 = red[3][k0];
        for (int k = k0 + 1; k < k0 + WPS; ++k) {
            sx0 = min(sx0, red[0][k]);
            sx1 = max(sx1, red[1][k]);
            sy0 = min(sy0, red[2][k]);
            sy1 = max(sy1, red[3][k]);
        }
        uint64_t* b = w.bbox + 4 * ((int64_t)blockIdx.x * (SY_TS / SY_SUB) + threadIdx.x);
        b[0] = sx0;
        b[1] = sx1;
        b[2] = sy0;
        b[3] = sy1;
    }
    if (threadIdx.x == 0) {
        for (int k = 1; k < SY_TS / 32; ++k) {
            amin = min(amin, red[4][k]);
            amax = max(amax, red[5][k]);
        }
        w.tile_a[blockIdx.x] = amin == amax ? bits_to_double(amin) : __longlong_as_double(0x7ff8000000000000ll);
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

// the FAST-SYM setup's per-particle passes fused: the sort-cell count of
// k_sort_count (alpha group, Morton cell) and the tie-bucket counts of
// k_tie_count in one pass; the two scatters in another
__global__ void k_sym_count(const double* __restrict__ pos, const double* __restrict__ alpha, int64_t n, double L,
                            SortWs sw, SymWs w) {
    const int G = 1 << sw.grid_log2;
    const double inv = (double)G / L;
    const double a_ref = alpha[0];
    const int64_t B = sym_tie_buckets(n);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = pos[2 * i], y = pos[2 * i + 1];
        int cx = (int)(x * inv), cy = (int)(y * inv);
        cx = cx < 0 ? 0 : (cx >= G ? G - 1 : cx);
        cy = cy < 0 ? 0 : (cy >= G ? G - 1 : cy);
        const int c = (int)morton2((uint32_t)cx, (uint32_t)cy) + (!(alpha[i] == a_ref) ? G * G : 0);
        sw.cell_of[i] = c;
        atomicAdd(&sw.cell_off[c], 1);
        atomicAdd(&w.tcnt[tie_bucket(x, L, B)], 1);
        atomicAdd(&w.tcnt[B + tie_bucket(y, L, B)], 1);
    }
}

__global__ void k_sym_scatter(const double* __restrict__ pos, int64_t n, double L, SortWs sw, SymWs w) {
    const int64_t B = sym_tie_buckets(n);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = sw.cell_of[i];
        sw.order[sw.cell_off[c] + atomicAdd(&sw.cell_cur[c], 1)] = (int32_t)i;
        const double x = pos[2 * i], y = pos[2 * i + 1];
        const int64_t bx = tie_bucket(x, L, B), by = B + tie_bucket(y, L, B);
        w.tval[w.tcnt[bx] + atomicAdd(&w.tcur[bx], 1)] = x;
        w.tval[w.tcnt[by] + atomicAdd(&w.tcur[by], 1)] = y;
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

// Per (warp, tile) image mode:
//   UNIFORM -- no receiver breakpoint inside or near the tile's box: one
//              image shift per receiver for the whole tile, d_src = d;
//   SEL     -- a breakpoint inside the box on axis x (SEL_X), y (SEL_Y) or
//              both, none near a source: per-pair image on that axis from
//              the breakpoint (an integer compare of the coordinate bits;
//              the > T image is the <= T one + L), d_src = d;
//   EDGE    -- a breakpoint within eps of the box: per-pair image and d_src
//              from the exact min-image arithmetic of the source side (the
//              reference's two directions of a pair whose fl(d / L) is within
//              ulps of +-1/2 do not use mirror images, e.g. lattice pairs
//              exactly L/2 apart);
//   GENERIC -- exact min-image arithmetic on both sides (receivers within
//              ulps of L/2 have ambiguous breakpoints; essentially never).
enum { SY_UNIFORM = 0, SY_SEL_X = 1, SY_SEL_Y = 2, SY_SEL_XY = 3, SY_EDGE_M = 4, SY_GENERIC = 5 };

// raw receiver coordinate from its selector: one of the two shifted copies is unshifted
BD_DEV double raw_coord(double c_le, double c_gt, double L) { return c_gt < L ? c_gt : c_le; }

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

// Same for 4 values: lane l holds the partial of source u ^ g4(l),
// g4(l) = (l >> 3) & 3; 6 shuffles + 6 adds for 4 sums.  Half the loop body
// of the 8-source groups (the hot loops then fit the small instruction
// caches better), 0.19 more adds per pair.
BD_DEV double tree4(const double v[4]) {
    double h[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) h[j] = v[j] + __shfl_xor_sync(0xffffffffu, v[j + 2], 16);
    double r = h[0] + __shfl_xor_sync(0xffffffffu, h[1], 8);
    r += __shfl_xor_sync(0xffffffffu, r, 4);
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    return r;
}

#ifndef BD_SY_G
#define BD_SY_G 4
#endif
#ifndef BD_SY_SELAXES
#define BD_SY_SELAXES 1
#endif
constexpr int SY_G = BD_SY_G;  // sources per transposed reduction (8 or 4)
static_assert(SY_G == 8 || SY_G == 4, "tree8 / tree4");
constexpr int SY_GSH = SY_G == 8 ? 2 : 3;  // lane bits below the source index of the transposed tree
BD_DEV double treeG(const double* v) { return SY_G == 8 ? tree8(v) : tree4(v); }

// Receiver data of one pass over a tile (NR of the lane's SY_R receivers):
// only what the pass's image mode needs is held in registers, loaded from the
// selector table (L1-resident) at the start of the pass.  The lane's
// receiver-side sums of the tile accumulate in sx / sy and are added to the
// lane's running totals (shared memory) at the end of the pass.
template <int MODE, int NR>
struct PassRecv {
    static constexpr bool PX = MODE >= SY_EDGE_M || (MODE & SY_SEL_X);  // per-pair x image
    static constexpr bool PY = MODE >= SY_EDGE_M || (MODE & SY_SEL_Y);
    static constexpr bool RAW = MODE >= SY_EDGE_M;  // both shifted copies (exact min image arithmetic)
    double cx[NR], cy[NR];  // the tile's image (uniform axis) or the <= T copy (per-pair axis)
    double gx[RAW ? NR : 1], gy[RAW ? NR : 1];  // the > T copy (EDGE / GENERIC)
    uint64_t Tx[PX && !RAW ? NR : 1], Ty[PY && !RAW ? NR : 1];
    double sx[NR], sy[NR];
};

// one source against the pass's receivers.  Receiver side: s{x,y} += alpha_k w d
// (FACT: w d, the tile's alpha applied at the end); source side: returns
// sum_m alpha_m w d_src (FACT: w d_src, the warp's alpha applied after the
// warp reduction) in bx / by.
template <int MODE, bool FACT, int NR>
BD_DEV void sym_pair(PassRecv<MODE, NR>& r, double sxv, double syv, double sav, const double* ra, double L,
                     double lo, double hi, double& bx, double& by) {
    using PR = PassRecv<MODE, NR>;
    bx = 0.0;
    by = 0.0;
    const uint64_t bsx = dbits(sxv), bsy = dbits(syv);
#pragma unroll
    for (int m = 0; m < NR; ++m) {
        double dx, dy, sxm, sym;
        if (PR::RAW) {
            // the receiver side's exact image (mi_fast is the reference's rule for |d| < L)
            dx = mi_fast(raw_coord(r.cx[m], r.gx[m], L) - sxv, L, lo, hi);
            dy = mi_fast(raw_coord(r.cy[m], r.gy[m], L) - syv, L, lo, hi);
            // the source side's own exact image
            sxm = -mi_fast(sxv - raw_coord(r.cx[m], r.gx[m], L), L, lo, hi);
            sym = -mi_fast(syv - raw_coord(r.cy[m], r.gy[m], L), L, lo, hi);
        } else {
            dx = r.cx[m] - sxv;
            dy = r.cy[m] - syv;
            if (PR::PX) dx = bsx > r.Tx[m] ? dx + L : dx;
            if (PR::PY) dy = bsy > r.Ty[m] ? dy + L : dy;
            sxm = dx;
            sym = dy;
        }
        const double w = inv_r3(fma(dx, dx, dy * dy));
        if (FACT) {
            r.sx[m] = fma(w, dx, r.sx[m]);
            r.sy[m] = fma(w, dy, r.sy[m]);
            bx = fma(w, sxm, bx);
            by = fma(w, sym, by);
        } else {
            const double ta = sav * w;
            r.sx[m] = fma(ta, dx, r.sx[m]);
            r.sy[m] = fma(ta, dy, r.sy[m]);
            const double tb = ra[m] * w;
            bx = fma(tb, sxm, bx);
            by = fma(tb, sym, by);
        }
    }
}

// per-lane running receiver sums A (ax, ay of SY_R receivers) in shared memory
struct LaneAcc {
    double* p;  // [SY_R][2][SY_CT] (this thread's column)
    BD_DEV double& ax(int m) const { return p[(2 * m) * SY_CT]; }
    BD_DEV double& ay(int m) const { return p[(2 * m + 1) * SY_CT]; }
};

// a shared-memory stage of source tile: positions and alphas
struct SymStage {
    const SymXY* xy;
    const double* a;
};

// One pass of the tile's `cnt` sources over receivers [M0, M0 + NR) of the
// lane.  Source side: the warp sums over those receivers go to
// bws[2 j .. 2 j + 1] (FIRST) or are added to them (later passes; the same
// lane owns the same entries in every pass, so the order is fixed).
// ta = the tile's alpha, wa = the warp's receiver alpha (FACT).
template <int MODE, bool FACT, int M0, int NR, bool FIRST>
BD_DEV void sym_pass(const SymWs& w, const int64_t* slot, const bool* act, double shx, double shy,
                     const SymStage& sm, int cnt, double L, double lo, double hi, double* bws, int lane, double ta,
                     double wa, const LaneAcc& acc) {
    using PR = PassRecv<MODE, NR>;
    PR r;
    double ra[FACT ? 1 : NR];
#pragma unroll
    for (int m = 0; m < NR; ++m) {
        r.sx[m] = 0.0;
        r.sy[m] = 0.0;
        if (PR::RAW) {
            const SelS q = w.sel[slot[M0 + m]];
            r.cx[m] = q.cx_le;
            r.gx[m] = q.cx_gt;
            r.cy[m] = q.cy_le;
            r.gy[m] = q.cy_gt;
        } else {
            // uniform axis: the receiver's raw coordinate minus the warp's image shift n L
            const SymXY p = (PR::PX && PR::PY) ? SymXY{0.0, 0.0} : w.sxy[slot[M0 + m]];
            if (PR::PX) {
                const SelS* q = w.sel + slot[M0 + m];
                r.cx[m] = q->cx_le;
                r.Tx[m] = q->Tx;
            } else {
                r.cx[m] = p.x - shx;
            }
            if (PR::PY) {
                const SelS* q = w.sel + slot[M0 + m];
                r.cy[m] = q->cy_le;
                r.Ty[m] = q->Ty;
            } else {
                r.cy[m] = p.y - shy;
            }
        }
        if (!FACT) ra[m] = act[M0 + m] ? w.sa[slot[M0 + m]] : 0.0;
    }
    int j = 0;
    const int g = (lane >> SY_GSH) & (SY_G - 1);  // this lane visits source j + (u ^ g) at step u
    for (; j + SY_G <= cnt; j += SY_G) {
        double bx[SY_G], by[SY_G];
#pragma unroll
        for (int u = 0; u < SY_G; ++u) {
            const SymXY p = sm.xy[j + (u ^ g)];
            sym_pair<MODE, FACT, NR>(r, p.x, p.y, FACT ? 0.0 : sm.a[j + (u ^ g)], ra, L, lo, hi, bx[u], by[u]);
        }
        double sx = treeG(bx), sy = treeG(by);
        if (FACT) {
            sx *= wa;
            sy *= wa;
        }
        if ((lane & ((1 << SY_GSH) - 1)) == 0) {
            const int k = j + g;
            bws[2 * k] = FIRST ? sx : bws[2 * k] + sx;
            bws[2 * k + 1] = FIRST ? sy : bws[2 * k + 1] + sy;
        }
    }
    for (; j < cnt; ++j) {
        double bx, by;
        const SymXY p = sm.xy[j];
        sym_pair<MODE, FACT, NR>(r, p.x, p.y, FACT ? 0.0 : sm.a[j], ra, L, lo, hi, bx, by);
        double sx = warp_sum(bx), sy = warp_sum(by);
        if (FACT) {
            sx *= wa;
            sy *= wa;
        }
        if (lane == 0) {
            bws[2 * j] = FIRST ? sx : bws[2 * j] + sx;
            bws[2 * j + 1] = FIRST ? sy : bws[2 * j + 1] + sy;
        }
    }
    const double f = FACT ? ta : 1.0;
#pragma unroll
    for (int m = 0; m < NR; ++m) {
        acc.ax(M0 + m) = fma(f, r.sx[m], acc.ax(M0 + m));
        acc.ay(M0 + m) = fma(f, r.sy[m], acc.ay(M0 + m));
    }
}

// the exact min-image modes: one pass per receiver (M0 = 0 .. SY_R - 1)
template <int MODE, bool FACT, int M0>
BD_DEV void sym_pass_each(const SymWs& w, const int64_t* slot, const bool* act, double shx, double shy,
                          const SymStage& sm, int cnt, double L, double lo, double hi, double* bws, int lane,
                          double ta, double wa, const LaneAcc& acc) {
    sym_pass<MODE, FACT, M0, 1, M0 == 0>(w, slot, act, shx, shy, sm, cnt, L, lo, hi, bws, lane, ta, wa, acc);
    if constexpr (M0 + 1 < SY_R)
        sym_pass_each<MODE, FACT, M0 + 1>(w, slot, act, shx, shy, sm, cnt, L, lo, hi, bws, lane, ta, wa, acc);
}

// a tile in mode MODE: one pass over all SY_R receivers, except the exact
// min-image modes (two copies per receiver and axis: passes of one receiver)
template <int MODE, bool FACT>
BD_DEV void sym_tile(const SymWs& w, const int64_t* slot, const bool* act, double shx, double shy,
                     const SymStage& sm, int cnt, double L, double lo, double hi, double* bws, int lane, double ta,
                     double wa, const LaneAcc& acc) {
    if (MODE < SY_EDGE_M) {
        sym_pass<MODE, FACT, 0, SY_R, true>(w, slot, act, shx, shy, sm, cnt, L, lo, hi, bws, lane, ta, wa, acc);
    } else {
        sym_pass_each<MODE, FACT, 0>(w, slot, act, shx, shy, sm, cnt, L, lo, hi, bws, lane, ta, wa, acc);
    }
}

// diagonal block (J == I): directed pairs, receiver side only, k != i
template <bool GEN>
BD_DEV void sym_diag(const SymWs& w, const int64_t* slot, const SymStage& sm, int cnt, int64_t base, double L,
                     double lo, double hi, const LaneAcc& acc) {
#pragma unroll
    for (int m = 0; m < SY_R; ++m) {
        const SelS q = w.sel[slot[m]];
        double ax = 0.0, ay = 0.0;
        for (int j = 0; j < cnt; ++j) {
            const SymXY p = sm.xy[j];
            double dx, dy;
            if (GEN) {
                dx = mi_fast(raw_coord(q.cx_le, q.cx_gt, L) - p.x, L, lo, hi);
                dy = mi_fast(raw_coord(q.cy_le, q.cy_gt, L) - p.y, L, lo, hi);
            } else {
                dx = (dbits(p.x) <= q.Tx ? q.cx_le : q.cx_gt) - p.x;
                dy = (dbits(p.y) <= q.Ty ? q.cy_le : q.cy_gt) - p.y;
            }
            double ta = sm.a[j] * inv_r3(fma(dx, dx, dy * dy));
            ta = base + j == slot[m] ? 0.0 : ta;
            ax = fma(ta, dx, ax);
            ay = fma(ta, dy, ay);
        }
        acc.ax(m) += ax;
        acc.ay(m) += ay;
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

BD_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr int SY_NW2 = SY_CT / 32;   // warps per CTA
#ifndef BD_SY_NS
#define BD_SY_NS 2
#endif
constexpr int SY_NS = BD_SY_NS;      // source stages
// dynamic smem per stage: positions (16 B) + alphas (8 B) of SY_TS sources,
// the warps' source-side sums (16 B per source and warp); + the lanes' receiver sums
#ifndef BD_SY_NBW
#define BD_SY_NBW 1
#endif
constexpr int SY_NBW = BD_SY_NBW;  // warp-sum buffers: one per stage, or one shared (+ a barrier per tile)
constexpr int SY_STAGE = SY_TS * 24;
constexpr int SY_BWS = SY_NW2 * SY_TS * 16;
constexpr int SY_SMEM = SY_NS * SY_STAGE + SY_NBW * SY_BWS + SY_R * 2 * SY_CT * 8;

// TMA of source tile t (SY_TS slots; fewer or none past n) into stage st
BD_DEV void sym_issue(const SymWs& w, int64_t n, int64_t t, unsigned char* smem, uint64_t* bars, int st) {
    const int64_t cnt = (t + 1) * SY_TS <= n ? SY_TS : (t * SY_TS < n ? n - t * SY_TS : 0);
    unsigned char* stg = smem + (size_t)st * SY_STAGE;
    // bulk copies move multiples of 16 bytes: an odd count of alphas reads one
    // more (never used; sa is padded to 256 bytes)
    const uint32_t ab = (uint32_t)((cnt * 8 + 15) / 16 * 16);
    mbar_expect_tx(&bars[st], (uint32_t)(cnt * 16) + ab);
    if (cnt) {
        bulk_g2s(stg, w.sxy + t * SY_TS, (uint32_t)(cnt * 16), &bars[st]);
        bulk_g2s(stg + SY_TS * 16, w.sa + t * SY_TS, ab, &bars[st]);
    }
}

// grid (Mb, 1 + chunks), SY_CT threads.  CTA (x, y): receiver block I = x;
// y = chunks (the last row): the diagonal block J = I (directed, receiver
// side only) when I is in [i0, i1), else nothing; y < chunks: distance
// chunk c = chunk0 + y cstep.  The diagonal row's short CTAs come last and
// fill the final wave.  Warp v of block I owns slots
// I*SY_BT + 32 SY_R v + lane + 32 m, m < SY_R.  Its receiver sums over the
// chunk go to apart[c]; the CTA's source-side sums of each tile of block
// J = I + d go to bpart[d - 1].  A CTA barrier ends every tile; the stage
// is then refilled (TMA) with the tile two ahead while the CTA adds its
// warps' source-side sums.  (Measured and dropped: decoupled warps with a
// per-stage ticket, the last warp summing and refilling -- 10.2 vs 9.5 ms at
// cfg3; persistent CTAs over an atomic work counter -- 9.7 vs 9.4 ms: the
// hot loop's code generation got worse.)
__global__ void __launch_bounds__(SY_CT, BD_SY_MINB) k_allpairs_sym(SymWs w, int64_t n, double L, double lo, double hi,
                                                                     int chunk0, int cstep, int64_t i0, int64_t i1) {
    extern __shared__ __align__(128) unsigned char sy_smem[];
    double* accs = reinterpret_cast<double*>(sy_smem + SY_NS * SY_STAGE + SY_NBW * SY_BWS);  // [SY_R][2][SY_CT]
    __shared__ __align__(8) uint64_t bars[SY_NS];
    __shared__ uint64_t wband[SY_NW2][2][4];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t Mb = sym_blocks(n), D = sym_D(n);
    const int64_t I = blockIdx.x;
#ifndef BD_SY_DIAG_LAST
#define BD_SY_DIAG_LAST 1
#endif
    // the diagonal row: last (its short CTAs fill the final wave: 9.13 ->
    // 9.11 ms at cfg3) or first (BD_SY_DIAG_LAST=0)
    const bool diag = BD_SY_DIAG_LAST ? blockIdx.y == gridDim.y - 1 : blockIdx.y == 0;
    if (diag && (I < i0 || I >= i1)) return;
    const int chunk = diag ? SY_S : chunk0 + ((int)blockIdx.y - (BD_SY_DIAG_LAST ? 0 : 1)) * cstep;
    const LaneAcc acc{accs + threadIdx.x};

    int64_t slot[SY_R];
    bool act[SY_R], amb = false;
    double ra0 = 0.0;
    bool wone = true;
#pragma unroll
    for (int m = 0; m < SY_R; ++m) {
        slot[m] = I * SY_BT + 32 * SY_R * wid + lane + 32 * m;
        act[m] = slot[m] < n;
        slot[m] = act[m] ? slot[m] : I * SY_BT;  // inactive lanes read a valid slot; their results are dropped
        amb |= act[m] && w.sel[slot[m]].amb;
        const double a = act[m] ? w.sa[slot[m]] : 0.0;
        if (m == 0) ra0 = a;
        acc.ax(m) = 0.0;
        acc.ay(m) = 0.0;
    }
    // The warp's breakpoint bands, per axis: receivers whose image flips from
    // n = +1 (s <= T) to 0 ("up", x_i above ~L/2) and from 0 to -1 (s > T,
    // "down"; also receivers without a breakpoint: n = 0 always).  A
    // sub-tile box [b0, b1] gives every receiver of the warp the same n when
    //   n =  0: b0 > max T_up and b1 <= min T_down
    //   n = +1: no down receiver and b1 <= min T_up
    //   n = -1: no up receiver and b0 > max T_down
    // and otherwise runs a per-pair image mode on that axis.
    uint64_t wb[2][4];  // [axis] {min T_up, max T_up, min T_down, max T_down}
    bool wtie = false;
#pragma unroll
    for (int ax = 0; ax < 2; ++ax) {
        wb[ax][0] = ~0ull;
        wb[ax][1] = 0;
        wb[ax][2] = ~0ull;
        wb[ax][3] = 0;
    }
#pragma unroll
    for (int m = 0; m < SY_R; ++m) {
        if (!act[m]) continue;
        const SelS q = w.sel[slot[m]];
        const uint64_t T[2] = {q.Tx, q.Ty};
        const bool up[2] = {q.cx_gt < L, q.cy_gt < L};
#pragma unroll
        for (int ax = 0; ax < 2; ++ax) {
            const int o = up[ax] && T[ax] != ~0ull ? 0 : 2;
            wb[ax][o] = min(wb[ax][o], T[ax]);
            wb[ax][o + 1] = max(wb[ax][o + 1], T[ax]);
        }
        wtie |= q.tie != 0;
    }
#pragma unroll
    for (int ax = 0; ax < 2; ++ax)
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            wb[ax][0] = min(wb[ax][0], (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)wb[ax][0], o));
            wb[ax][1] = max(wb[ax][1], (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)wb[ax][1], o));
            wb[ax][2] = min(wb[ax][2], (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)wb[ax][2], o));
            wb[ax][3] = max(wb[ax][3], (uint64_t)__shfl_xor_sync(0xffffffffu, (unsigned long long)wb[ax][3], o));
        }
    wtie = __any_sync(0xffffffffu, wtie);
    if (lane == 0) {
#pragma unroll
        for (int ax = 0; ax < 2; ++ax)
#pragma unroll
            for (int k = 0; k < 4; ++k) wband[wid][ax][k] = wb[ax][k];
    }
    // the warp's receivers all active with one alpha: factored tiles possible
    const double wa = __shfl_sync(0xffffffffu, ra0, 0);
#pragma unroll
    for (int m = 0; m < SY_R; ++m) wone &= act[m] && (act[m] ? w.sa[slot[m]] : 0.0) == wa;
    const bool wfact = __all_sync(0xffffffffu, wone);

    // this CTA's distances [d0, d1): chunk c covers [1 + c per, 1 + (c + 1) per) of [1, D]
    const int64_t per = sym_per(n);
    int64_t d0, d1;
    if (diag) {
        d0 = 0;
        d1 = 1;
    } else {
        d0 = 1 + (int64_t)chunk * per < D + 1 ? 1 + (int64_t)chunk * per : D + 1;
        d1 = 1 + ((int64_t)chunk + 1) * per < D + 1 ? 1 + ((int64_t)chunk + 1) * per : D + 1;
    }
    const bool even = (Mb & 1) == 0;
    constexpr int64_t tpb = SY_BT / SY_TS;  // source tiles per block
    const int64_t nq = d1 > d0 ? (d1 - d0) * tpb : 0;

    if (threadIdx.x == 0) {
        for (int k = 0; k < SY_NS; ++k) mbar_init(&bars[k], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const bool wamb = __any_sync(0xffffffffu, amb);
    if (threadIdx.x == 0)
        for (int64_t qi = 0; qi < SY_NS && qi < nq; ++qi)
            sym_issue(w, n, ((I + d0 + qi / tpb) % Mb) * tpb + qi % tpb, sy_smem, bars, (int)qi);

    for (int64_t qi = 0; qi < nq; ++qi) {
        const int st = (int)(qi % SY_NS);
        const int64_t d = d0 + qi / tpb;
        const int64_t J = (I + d) % Mb;
        const int64_t t = J * tpb + qi % tpb;
        const int64_t base = t * SY_TS;
        const int cnt = (int)((t + 1) * SY_TS <= n ? SY_TS : (base < n ? n - base : 0));
        const bool use = !(even && d == D && d > 0 && I >= Mb / 2) && cnt > 0;
        unsigned char* stg = sy_smem + (size_t)st * SY_STAGE;
        const SymStage sm{reinterpret_cast<const SymXY*>(stg), reinterpret_cast<const double*>(stg + SY_TS * 16)};
        double* bw = reinterpret_cast<double*>(sy_smem + SY_NS * SY_STAGE + (st % SY_NBW) * SY_BWS);  // [NW2][TS][2]
        double* bws = bw + (size_t)wid * SY_TS * 2;
        mbar_wait(&bars[st], (uint32_t)((qi / SY_NS) & 1));
        if (use && d == 0) {
            if (wamb)
                sym_diag<true>(w, slot, sm, cnt, base, L, lo, hi, acc);
            else
                sym_diag<false>(w, slot, sm, cnt, base, L, lo, hi, acc);
        } else if (use) {
            const double ta = w.tile_a[t];
            const bool fact = wfact && ta == ta;  // NaN: mixed tile
            const double eps = sym_tie_eps(L);    // >> the ulps of L in which image ties live
            for (int sub = 0; sub * SY_SUB < cnt; ++sub) {
                const int c0 = sub * SY_SUB;
                const int cs = cnt - c0 < SY_SUB ? cnt - c0 : SY_SUB;
                const uint64_t* bb = w.bbox + 4 * (t * (SY_TS / SY_SUB) + sub);
                // the image mode of this sub-tile: per axis a warp-uniform shift n or per-pair
                int nimg[2], sel = 0;
#pragma unroll
                for (int ax = 0; ax < 2; ++ax) {
                    const uint64_t b0 = bb[2 * ax], b1 = bb[2 * ax + 1];
                    const uint64_t mnu = wband[wid][ax][0], mxu = wband[wid][ax][1];
                    const uint64_t mnd = wband[wid][ax][2], mxd = wband[wid][ax][3];
                    const bool has_up = mxu >= mnu, has_dn = mxd >= mnd;
                    if ((!has_up || b0 > mxu) && (!has_dn || b1 <= mnd)) {
                        nimg[ax] = 0;
                    } else if (!has_dn && b1 <= mnu) {
                        nimg[ax] = 1;
                    } else if (!has_up && b0 > mxd) {
                        nimg[ax] = -1;
                    } else {
                        nimg[ax] = 0;
                        sel |= ax == 0 ? SY_SEL_X : SY_SEL_Y;
                    }
                }
                const double shx = (double)nimg[0] * L, shy = (double)nimg[1] * L;
                bool any_edge = false;
                if (wtie) {  // lattice-like states only: a receiver with a source within eps of its breakpoint
                    bool edge = false;
#pragma unroll
                    for (int m = 0; m < SY_R; ++m) {
                        const SelS q = w.sel[slot[m]];
                        edge |= act[m] && (((q.tie & 1) && near_window(bb[0], bb[1], q.Tx, eps)) ||
                                           ((q.tie & 2) && near_window(bb[2], bb[3], q.Ty, eps)));
                    }
                    any_edge = __any_sync(0xffffffffu, edge);
                }
                const SymStage ss{sm.xy + c0, sm.a + c0};
                double* bs = bws + 2 * c0;
                if (wamb) {
                    sym_tile<SY_GENERIC, false>(w, slot, act, shx, shy, ss, cs, L, lo, hi, bs, lane, ta, wa, acc);
                } else if (any_edge) {
                    sym_tile<SY_EDGE_M, false>(w, slot, act, shx, shy, ss, cs, L, lo, hi, bs, lane, ta, wa, acc);
                } else if (fact) {
#if !BD_SY_SELAXES
                    if (sel) sel = SY_SEL_XY;  // one per-pair loop for both axes: less hot code
#endif
                    switch (sel) {
                        case 0: sym_tile<SY_UNIFORM, true>(w, slot, act, shx, shy, ss, cs, L, lo, hi, bs, lane, ta, wa, acc); break;
                        case SY_SEL_X: sym_tile<SY_SEL_X, true>(w, slot, act, shx, shy, ss, cs, L, lo, hi, bs, lane, ta, wa, acc); break;
                        case SY_SEL_Y: sym_tile<SY_SEL_Y, true>(w, slot, act, shx, shy, ss, cs, L, lo, hi, bs, lane, ta, wa, acc); break;
                        default: sym_tile<SY_SEL_XY, true>(w, slot, act, shx, shy, ss, cs, L, lo, hi, bs, lane, ta, wa, acc); break;
                    }
                } else {
                    if (sel == 0)
                        sym_tile<SY_UNIFORM, false>(w, slot, act, shx, shy, ss, cs, L, lo, hi, bs, lane, ta, wa, acc);
                    else
                        sym_tile<SY_SEL_XY, false>(w, slot, act, shx, shy, ss, cs, L, lo, hi, bs, lane, ta, wa, acc);
                }
            }
        }
        __syncthreads();  // stage st consumed; the warps' source-side sums of tile qi complete
        if (threadIdx.x == 0 && qi + SY_NS < nq) {
            fence_proxy_async_smem();
            sym_issue(w, n, ((I + d0 + (qi + SY_NS) / tpb) % Mb) * tpb + (qi + SY_NS) % tpb, sy_smem, bars, st);
        }
        if (use && d > 0) {
            // CTA sum of the warp sums (warp order) -> one partial per (d, source); the refill
            // writes only the stage's source arrays, not these sums (read before the next barrier)
            for (int e = threadIdx.x; e < 2 * cnt; e += SY_CT) {
                double v = 0.0;
#pragma unroll
                for (int ww = 0; ww < SY_NW2; ++ww) v += bw[(size_t)ww * SY_TS * 2 + e];
                w.bpart[(size_t)(d - 1) * n * 2 + (size_t)base * 2 + e] = v;
            }
        }
        if (SY_NBW == 1) __syncthreads();  // the shared warp-sum buffer is written again by the next tile
    }
#pragma unroll
    for (int m = 0; m < SY_R; ++m) {
        if (!act[m]) continue;
        w.apart[(size_t)chunk * n * 2 + 2 * slot[m]] = acc.ax(m);
        w.apart[(size_t)chunk * n * 2 + 2 * slot[m] + 1] = acc.ay(m);
    }
}

// P = A - B per slot over this rank's chunks / distances / diagonal blocks, fixed order -> part (n, 2)
__global__ void k_sym_partial(int64_t n, SymWs w, SymRange g, double* __restrict__ part) {
    const int64_t Mb = sym_blocks(n), D = sym_D(n), per = sym_per(n);
    const bool even = (Mb & 1) == 0;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        // 16-byte loads, the sums in a fixed order: this rank's chunks ascending, the
        // diagonal block, then the source-side distances of those chunks ascending
        double ax = 0.0, ay = 0.0, bx = 0.0, by = 0.0;
        const double2* ap = reinterpret_cast<const double2*>(w.apart) + s;
#pragma unroll 8
        for (int k = 0; k < g.nch; ++k) {
            const double2 v = __ldcs(ap + (size_t)(g.c0 + k * g.cs) * n);
            ax += v.x;
            ay += v.y;
        }
        const int64_t J = s / SY_BT;
        if (J >= g.i0 && J < g.i1) {
            const double2 v = __ldcs(ap + (size_t)SY_S * n);
            ax += v.x;
            ay += v.y;
        }
        // d = D of an even block count belongs to the lower block only
        const bool skipD = even && (J - D + Mb) % Mb >= Mb / 2;
        const double2* bp = reinterpret_cast<const double2*>(w.bpart) + s;
        // the distances of this rank's chunks in ascending order as one flat
        // loop (independent loads in flight; the same addition order)
        const int64_t dmax = skipD ? D - 1 : D;
        const int per32 = (int)per, nf = g.nch * per32;
#pragma unroll 8
        for (int f = 0; f < nf; ++f) {
            const int q = f / per32;
            const int64_t c = g.c0 + (int64_t)q * g.cs;
            const int64_t d = 1 + c * per + (f - q * per32);
            if (d <= dmax) {
                const double2 v = __ldcs(bp + (size_t)(d - 1) * n);
                bx += v.x;
                by += v.y;
            }
        }
        part[2 * s] = ax - bx;
        part[2 * s + 1] = ay - by;
    }
}

// F = mu P per slot, written in particle order (out, err: 0, or -1 = re-scan exactly)
__global__ void k_sym_finish(int64_t n, SymWs w, const double* __restrict__ part, double* __restrict__ out,
                             int64_t* __restrict__ err) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const double mu = w.smu[s];
        const double fx = mu * part[2 * s], fy = mu * part[2 * s + 1];
        const int64_t i = w.sort.order[s];
        out[2 * i] = fx;
        out[2 * i + 1] = fy;
        err[i] = (isfinite(fx) && isfinite(fy)) ? 0 : -1;
    }
}

#endif  // __CUDACC__

BD_HD SymRange sym_range(int64_t n, int rank, int world) {
    // chunks dealt round-robin: every rank gets near and far block distances
    // alike (the per-pair image modes cluster at some distances), and the
    // half-weight last distance (d = D for even Mb) lands on one rank only
    SymRange g;
    const int64_t S = sym_chunks(n), Mb = sym_blocks(n);
    g.c0 = rank;
    g.cs = world;
    g.nch = (sym_D(n) > 0 && rank < S) ? (int)((S - 1 - rank) / world + 1) : 0;  // no chunks without block pairs
    g.i0 = (int64_t)rank * Mb / world;
    g.i1 = (int64_t)(rank + 1) * Mb / world;
    return g;
}

}  // namespace bd
