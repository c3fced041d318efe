// bd_allpairs_fast.cuh -- FAST all-pairs force: spatially sorted, tile-uniform images.
//
// Same force as _kernels.long_range_kernel (_kernels.py:26-59) to ~1e-13
// relative per particle, restructured so that the FP64 pipe does nothing but
// the force arithmetic (12 FP64 instructions per pair):
//
//  1. every step the particles are counting-sorted into Morton order of a
//     power-of-two cell grid (deterministic: ties by particle index), and
//     packed as 48-byte source records {x, y, a, 1.5a, 1.875a, mu} in that
//     order, with the x/y bounding box (as bit patterns) of every tile of
//     FS_TS consecutive sources;
//  2. receivers are the same sorted slots, so a warp's 32 receivers and a
//     source tile are both compact blobs.  For a (warp, tile) pair whose
//     boxes lie on one side of every receiver's exact image breakpoint
//     (axis_select, bd_allpairs.cuh) the minimum-image shift is a per-thread
//     constant for the whole tile -> no per-pair image work at all; other
//     (warp, tile) pairs fall back to the per-pair integer select;
//  3. r^-3 = y0^3 (1 - e)^(-3/2), y0 = MUFU.RSQ64H(r2), e = 1 - r2 y0^2,
//     expanded to second order with the per-source constants
//     (a, 1.5a, 1.875a): s = y0^3 (a + e (1.5a + 1.875a e)) -- 6 FP64
//     instructions, truncation error ~2e0^3 (e0 ~ 2^-20) ~ 1e-18;
//  4. results are written per sorted slot (contiguous -- the unit the
//     multi-GPU all-gather moves) and scattered back to particle order.
#pragma once

#include "bd_allpairs.cuh"
#include "bd_exec.cuh"

namespace bd {

struct alignas(16) Src6 {
    double x, y, a0, a1, a2, mu;
};

constexpr int FS_BT = 128;  // threads per CTA (4 warps; FS_R receivers each)
constexpr int FS_TS = 256;  // sources per smem stage (12 KiB)

struct SortWs {
    int32_t* cell_of;   // (n) Morton cell of each particle
    int32_t* cell_off;  // (ncells + 1) counts -> offsets
    int32_t* cell_cur;  // (ncells) scatter cursors
    int32_t* order;     // (n) sorted slot -> particle
    Src6* src;          // (n) packed sources in slot order
    uint64_t* bbox;     // (ntiles, 4) min/max bits of x and y per tile
    double* slot3;      // (n, 3) per slot: fx, fy, flag (0 ok / -1 exact re-scan)
    double* part3;      // (splits, n, 3) per source partition: partial fx, fy, flag
    int32_t grid_log2;  // cells per axis = 2^grid_log2
    int32_t splits;     // source partitions per receiver (fast_splits)
};

// Source partitions per receiver, a function of n ONLY (never of the GPU
// count, so sharded results stay bit-identical for every world size): enough
// (receiver, partition) work items for a full occupancy wave on one B200
// even when 8 ranks share the receivers; capped at 16 and at half the tiles.
BD_HD int fast_splits(int64_t n) {
    const int64_t tiles = (n + 255) / 256;
    int64_t s = 1;
    while (s < 16 && n * s < (int64_t)148 * 1024 * 8 && 2 * s <= tiles) s *= 2;
    return (int)s;
}

BD_HD int fast_grid_log2(int64_t n) {
    int g = 1;
    while ((int64_t)1 << (2 * g) < n / 2 && g < 15) ++g;  // ~2 particles per cell
    return g;
}

BD_HD int64_t fast_ncells(int64_t n) { return (int64_t)1 << (2 * fast_grid_log2(n)); }

BD_HD int64_t fs_align(int64_t x) { return (x + 255) & ~(int64_t)255; }

// bytes of the FAST-path scratch for n particles
BD_HD int64_t fast_ws_bytes(int64_t n) {
    const int64_t nc = fast_ncells(n), nt = (n + FS_TS - 1) / FS_TS;
    return fs_align(4 * n) + fs_align(4 * (2 * nc + 1)) + fs_align(8 * nc) + fs_align(4 * n) + fs_align(48 * n) +
           fs_align(32 * nt) + fs_align(24 * n) + fs_align(24 * n * fast_splits(n)) + 256;
}

BD_HD SortWs fast_ws_carve(void* base, int64_t n) {
    const int64_t nc = fast_ncells(n), nt = (n + FS_TS - 1) / FS_TS;
    char* b = (char*)(((uintptr_t)base + 255) & ~(uintptr_t)255);
    SortWs w;
    w.grid_log2 = fast_grid_log2(n);
    w.cell_of = (int32_t*)b; b += fs_align(4 * n);
    w.cell_off = (int32_t*)b; b += fs_align(4 * (2 * nc + 1));  // 2 nc: FAST-SYM sorts by (group, cell)
    w.cell_cur = (int32_t*)b; b += fs_align(8 * nc);
    w.order = (int32_t*)b; b += fs_align(4 * n);
    w.src = (Src6*)b; b += fs_align(48 * n);
    w.bbox = (uint64_t*)b; b += fs_align(32 * nt);
    w.slot3 = (double*)b; b += fs_align(24 * n);
    w.part3 = (double*)b;
    w.splits = fast_splits(n);
    return w;
}

BD_HD uint32_t morton2(uint32_t x, uint32_t y) {
    auto spread = [](uint32_t v) {
        v &= 0xffff;
        v = (v | (v << 8)) & 0x00ff00ff;
        v = (v | (v << 4)) & 0x0f0f0f0f;
        v = (v | (v << 2)) & 0x33333333;
        v = (v | (v << 1)) & 0x55555555;
        return v;
    };
    return spread(x) | (spread(y) << 1);
}

#if defined(__CUDACC__)

// group_alpha (FAST-SYM): particles whose alpha differs from alpha[0] sort
// after all others -- cell keys c + G^2 -- so source tiles and receiver warps
// carry one alpha (bd_allpairs_sym.cuh, factored pair evaluation)
__global__ void k_sort_count(const double* __restrict__ pos, int64_t n, double L, SortWs w,
                             const double* __restrict__ group_alpha = nullptr) {
    const int G = 1 << w.grid_log2;
    const double inv = (double)G / L;
    const double a_ref = group_alpha ? group_alpha[0] : 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int cx = (int)(pos[2 * i] * inv), cy = (int)(pos[2 * i + 1] * inv);
        cx = cx < 0 ? 0 : (cx >= G ? G - 1 : cx);
        cy = cy < 0 ? 0 : (cy >= G ? G - 1 : cy);
        const int c = (int)morton2((uint32_t)cx, (uint32_t)cy) +
                      ((group_alpha && !(group_alpha[i] == a_ref)) ? G * G : 0);
        w.cell_of[i] = c;
        atomicAdd(&w.cell_off[c], 1);
    }
}

// single-CTA exclusive scan of the cell counts: warp w owns a contiguous
// segment of the cells and walks it in coalesced 32-cell chunks (8 loads in
// flight); pass 1 sums the segments, one warp scans the 32 segment totals,
// pass 2 writes the offsets (and zeroes the scatter cursors)
__device__ void sort_scan_cta(SortWs w, int64_t ncells);

__global__ void __launch_bounds__(1024) k_sort_scan(SortWs w, int64_t ncells) { sort_scan_cta(w, ncells); }

// two independent scans in one launch: CTA 0 scans (w0, n0), CTA 1 (w1, n1)
__global__ void __launch_bounds__(1024) k_sort_scan2(SortWs w0, int64_t n0, SortWs w1, int64_t n1) {
    if (blockIdx.x == 0)
        sort_scan_cta(w0, n0);
    else
        sort_scan_cta(w1, n1);
}

__device__ void sort_scan_cta(SortWs w, int64_t ncells) {
    __shared__ int64_t seg[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t per = ((ncells + 31) / 32 + 31) & ~(int64_t)31;
    const int64_t c0 = wid * per, c1 = c0 + per < ncells ? c0 + per : ncells;
    int64_t sum = 0;
#pragma unroll 8
    for (int64_t c = c0 + lane; c < c1; c += 32) sum += w.cell_off[c];
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) seg[wid] = sum;
    __syncthreads();
    if (wid == 0) {
        const int64_t v = seg[lane];
        int64_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        seg[lane] = inc - v;
        if (lane == 31) w.cell_off[ncells] = (int32_t)inc;
    }
    __syncthreads();
    int64_t carry = seg[wid];
    // 8 chunks of 32 loaded before they are scanned (the carry chain would
    // otherwise serialise one global-load latency per chunk)
    for (int64_t base = c0; base < c1; base += 8 * 32) {
        int32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t c = base + 32 * u + lane;
            v[u] = c < c1 ? w.cell_off[c] : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t c = base + 32 * u + lane;
            int64_t inc = v[u];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            if (c < c1) {
                w.cell_off[c] = (int32_t)(carry + inc - v[u]);
                w.cell_cur[c] = 0;
            }
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
    }
}

__global__ void k_sort_scatter(int64_t n, SortWs w) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int c = w.cell_of[i];
        w.order[w.cell_off[c] + atomicAdd(&w.cell_cur[c], 1)] = (int32_t)i;
    }
}

// deterministic order inside each cell (ascending particle index)
__global__ void k_sort_fix(int64_t ncells, SortWs w) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncells; c += (int64_t)gridDim.x * blockDim.x) {
        int32_t* a = w.order + w.cell_off[c];
        const int32_t m = w.cell_off[c + 1] - w.cell_off[c];
        if (m <= 24) {  // the usual case: sort a private copy (one pass in, one out)
            int32_t v[24];
            for (int32_t j = 0; j < m; ++j) v[j] = a[j];
            for (int32_t j = 1; j < m; ++j) {
                const int32_t t = v[j];
                int32_t k = j - 1;
                while (k >= 0 && v[k] > t) {
                    v[k + 1] = v[k];
                    --k;
                }
                v[k + 1] = t;
            }
            for (int32_t j = 0; j < m; ++j) a[j] = v[j];
            continue;
        }
        for (int32_t j = 1; j < m; ++j) {
            const int32_t v = a[j];
            int32_t k = j - 1;
            while (k >= 0 && a[k] > v) {
                a[k + 1] = a[k];
                --k;
            }
            a[k + 1] = v;
        }
    }
}

// one CTA per tile of FS_TS slots: pack + tile bounding box
__global__ void __launch_bounds__(FS_TS) k_pack6(const double* __restrict__ pos, const double* __restrict__ alpha,
                                                 const double* __restrict__ mu, int64_t n, SortWs w) {
    __shared__ uint64_t red[4][FS_TS / 32];
    const int64_t s = (int64_t)blockIdx.x * FS_TS + threadIdx.x;
    uint64_t xmin = ~0ull, xmax = 0, ymin = ~0ull, ymax = 0;
    if (s < n) {
        const int64_t i = w.order[s];
        const double x = pos[2 * i], y = pos[2 * i + 1], a = alpha[i];
        Src6 r;
        r.x = x;
        r.y = y;
        r.a0 = a;
        r.a1 = 1.5 * a;
        r.a2 = 1.875 * a;
        r.mu = mu[i];
        w.src[s] = r;
        xmin = xmax = dbits(x);
        ymin = ymax = dbits(y);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        xmin = min(xmin, __shfl_xor_sync(0xffffffffu, xmin, o));
        xmax = max(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
        ymin = min(ymin, __shfl_xor_sync(0xffffffffu, ymin, o));
        ymax = max(ymax, __shfl_xor_sync(0xffffffffu, ymax, o));
    }
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        red[0][wid] = xmin;
        red[1][wid] = xmax;
        red[2][wid] = ymin;
        red[3][wid] = ymax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < FS_TS / 32; ++k) {
            xmin = min(xmin, red[0][k]);
            xmax = max(xmax, red[1][k]);
            ymin = min(ymin, red[2][k]);
            ymax = max(ymax, red[3][k]);
        }
        uint64_t* b = w.bbox + 4 * blockIdx.x;
        b[0] = xmin;
        b[1] = xmax;
        b[2] = ymin;
        b[3] = ymax;
    }
}

// R receivers per thread: each smem source is loaded once for R pair terms
// (halves LDS per pair at R = 2) and the R x unroll independent pair chains
// hide the FP64 / MUFU latencies.
template <int R>
struct RecvF {
    double cx_le[R], cx_gt[R], cy_le[R], cy_gt[R];
    uint64_t Tx[R], Ty[R];
    double fx[R], fy[R];
    int64_t slot[R];
};

template <int R, bool CHECK_SELF, bool SELECT>
BD_DEV void fast_term(RecvF<R>& r, const Src6& q, int64_t k, const double* cx, const double* cy) {
    const uint64_t qx = dbits(q.x), qy = dbits(q.y);
#pragma unroll
    for (int m = 0; m < R; ++m) {
        double ax = cx[m], ay = cy[m];
        if (SELECT) {
            ax = qx <= r.Tx[m] ? r.cx_le[m] : r.cx_gt[m];
            ay = qy <= r.Ty[m] ? r.cy_le[m] : r.cy_gt[m];
        }
        const double dx = ax - q.x, dy = ay - q.y;
        const double r2 = fma(dx, dx, dy * dy);
        const double y0 = rsqrt_mufu(r2);
        const double t = y0 * y0;
        const double e = fma(-r2, t, 1.0);
        const double y3 = t * y0;
        const double u = fma(fma(q.a2, e, q.a1), e, q.a0);
        double s = y3 * u;
        if (CHECK_SELF) s = (k == r.slot[m]) ? 0.0 : s;
        r.fx[m] = fma(s, dx, r.fx[m]);
        r.fy[m] = fma(s, dy, r.fy[m]);
    }
}

template <int R, bool CHECK_SELF, bool SELECT>
BD_DEV void fast_tile(RecvF<R>& r, const Src6* sm, int cnt, int64_t base, const double* cx, const double* cy) {
    if (cnt == FS_TS && !CHECK_SELF) {
#pragma unroll(8 / R)
        for (int j = 0; j < FS_TS; ++j) fast_term<R, false, SELECT>(r, sm[j], base + j, cx, cy);
    } else {
        for (int j = 0; j < cnt; ++j) fast_term<R, CHECK_SELF, SELECT>(r, sm[j], base + j, cx, cy);
    }
}

// receivers per thread: R = 2 (126 registers, 16 warps/SM) measured slower
// than R = 1 (64 registers, 32 warps/SM): 17.8 vs 16.7 ms at N = 131,072
constexpr int FS_R = 1;
constexpr int FS_RPB = FS_BT * FS_R;     // receivers per CTA

// receivers = sorted slots [i0, i1); CTA b owns [i0 + b*FS_RPB, +FS_RPB),
// thread t the slots t and t + FS_BT of it
__global__ void __launch_bounds__(FS_BT, 8)
    k_allpairs_fast(SortWs w, int64_t n, double L, double lo, double hi, int64_t i0, int64_t i1,
                    double* __restrict__ slot3) {
    __shared__ __align__(128) Src6 tile[2][FS_TS];
    __shared__ __align__(8) uint64_t bars[2];
    constexpr int R = FS_R;

    const int64_t rb0 = i0 + (int64_t)blockIdx.x * FS_RPB;
    const int64_t rb1 = rb0 + FS_RPB < i1 ? rb0 + FS_RPB : i1;
    RecvF<R> r;
    double mux[R], xs[R], ys[R];
    bool act[R], amb = false;
#pragma unroll
    for (int m = 0; m < R; ++m) {
        const int64_t slot = rb0 + threadIdx.x + m * FS_BT;
        act[m] = slot < rb1;
        const Src6 me = w.src[act[m] ? slot : rb0];
        r.slot[m] = act[m] ? slot : -1;
        r.fx[m] = 0.0;
        r.fy[m] = 0.0;
        const AxisSel sx = axis_select(me.x, L, lo, hi), sy = axis_select(me.y, L, lo, hi);
        r.Tx[m] = sx.T;
        r.Ty[m] = sy.T;
        r.cx_le[m] = me.x + sx.shift_le;
        r.cx_gt[m] = me.x + sx.shift_gt;
        r.cy_le[m] = me.y + sy.shift_le;
        r.cy_gt[m] = me.y + sy.shift_gt;
        mux[m] = me.mu;
        xs[m] = me.x;
        ys[m] = me.y;
        amb |= act[m] && (sx.amb || sy.amb);
    }
    const bool generic = __syncthreads_or(amb);
    int64_t e[R];
#pragma unroll
    for (int m = 0; m < R; ++m) e[m] = 0;

    // this CTA's source partition: tiles [tb, te) of the sorted sources
    const int64_t ntiles_all = (n + FS_TS - 1) / FS_TS;
    const int64_t per_part = (ntiles_all + gridDim.y - 1) / gridDim.y;
    const int64_t tb = (int64_t)blockIdx.y * per_part;
    const int64_t te = tb + per_part < ntiles_all ? tb + per_part : ntiles_all;
    const int64_t ntiles = te > tb ? te - tb : 0;
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int64_t u = 0; u < 2 && u < ntiles; ++u) {
            const int64_t t = tb + u;
            const int64_t cnt = (t + 1) * FS_TS <= n ? FS_TS : n - t * FS_TS;
            mbar_expect_tx(&bars[u], (uint32_t)(cnt * sizeof(Src6)));
            bulk_g2s(&tile[u][0], w.src + t * FS_TS, (uint32_t)(cnt * sizeof(Src6)), &bars[u]);
        }
    }
    for (int64_t u = 0; u < ntiles; ++u) {
        const int64_t t = tb + u;
        const int st = (int)(u & 1);
        const uint64_t* bb = w.bbox + 4 * t;
        const uint64_t bx0 = bb[0], bx1 = bb[1], by0 = bb[2], by1 = bb[3];
        mbar_wait(&bars[st], (uint32_t)((u >> 1) & 1));
        const Src6* sm = tile[st];
        const int64_t base = t * FS_TS;
        const int cnt = (int)((t + 1) * FS_TS <= n ? FS_TS : n - base);
        const bool diag = base < rb1 && base + cnt > rb0;
        if (generic) {
            for (int j = 0; j < cnt; ++j) {
                const int64_t k = base + j;
                const Src6 q = sm[j];
#pragma unroll
                for (int m = 0; m < R; ++m) {
                    if (k == r.slot[m]) continue;
                    const double dx = mi_fast(xs[m] - q.x, L, lo, hi), dy = mi_fast(ys[m] - q.y, L, lo, hi);
                    const double r2 = dx * dx + dy * dy;
                    if (dbits(r2) == 0ull) {
                        e[m] = -1;
                        continue;
                    }
                    const double wgt = q.a0 / (r2 * sqrt(r2));
                    r.fx[m] = fma(wgt, dx, r.fx[m]);
                    r.fy[m] = fma(wgt, dy, r.fy[m]);
                }
            }
        } else {
            // tile-uniform image shift of each receiver, if any
            double cx[R], cy[R];
            bool uni = true;
#pragma unroll
            for (int m = 0; m < R; ++m) {
                const bool xle = bx1 <= r.Tx[m], xgt = bx0 > r.Tx[m], yle = by1 <= r.Ty[m], ygt = by0 > r.Ty[m];
                uni &= !act[m] || ((xle || xgt) && (yle || ygt));
                cx[m] = xle ? r.cx_le[m] : r.cx_gt[m];
                cy[m] = yle ? r.cy_le[m] : r.cy_gt[m];
            }
            if (__all_sync(0xffffffffu, uni)) {
                if (diag) fast_tile<R, true, false>(r, sm, cnt, base, cx, cy);
                else fast_tile<R, false, false>(r, sm, cnt, base, cx, cy);
            } else {
                if (diag) fast_tile<R, true, true>(r, sm, cnt, base, cx, cy);
                else fast_tile<R, false, true>(r, sm, cnt, base, cx, cy);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && u + 2 < ntiles) {
            const int64_t t2 = t + 2;
            const int64_t cnt2 = (t2 + 1) * FS_TS <= n ? FS_TS : n - t2 * FS_TS;
            mbar_expect_tx(&bars[st], (uint32_t)(cnt2 * sizeof(Src6)));
            bulk_g2s(&tile[st][0], w.src + t2 * FS_TS, (uint32_t)(cnt2 * sizeof(Src6)), &bars[st]);
        }
    }
#pragma unroll
    for (int m = 0; m < R; ++m) {
        if (!act[m]) continue;
        const int64_t slot = r.slot[m];
        if (gridDim.y == 1) {
            const double fx = mux[m] * r.fx[m], fy = mux[m] * r.fy[m];
            slot3[3 * slot] = fx;
            slot3[3 * slot + 1] = fy;
            slot3[3 * slot + 2] = (isfinite(fx) && isfinite(fy) && e[m] == 0) ? 0.0 : -1.0;  // -1: exact re-scan
        } else {
            double* o = w.part3 + 3 * ((int64_t)blockIdx.y * n + slot);
            o[0] = r.fx[m];
            o[1] = r.fy[m];
            o[2] = e[m] == 0 ? 0.0 : -1.0;
        }
    }
}

// partial sums of the source partitions, added in partition order (deterministic)
__global__ void k_reduce_parts(int64_t s0, int64_t s1, int64_t n, SortWs w, double* __restrict__ slot3) {
    for (int64_t s = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < s1; s += (int64_t)gridDim.x * blockDim.x) {
        double fx = 0.0, fy = 0.0, flag = 0.0;
        for (int p = 0; p < w.splits; ++p) {
            const double* o = w.part3 + 3 * ((int64_t)p * n + s);
            fx += o[0];
            fy += o[1];
            flag = o[2] != 0.0 ? -1.0 : flag;
        }
        const double mu = w.src[s].mu;
        fx = mu * fx;
        fy = mu * fy;
        slot3[3 * s] = fx;
        slot3[3 * s + 1] = fy;
        slot3[3 * s + 2] = (isfinite(fx) && isfinite(fy) && flag == 0.0) ? 0.0 : -1.0;
    }
}

// slot results -> particle order
__global__ void k_unsort_forces(int64_t s0, int64_t s1, SortWs w, const double* __restrict__ slot3,
                                double* __restrict__ out, int64_t* __restrict__ err) {
    for (int64_t s = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < s1; s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = w.order[s];
        out[2 * i] = slot3[3 * s];
        out[2 * i + 1] = slot3[3 * s + 1];
        err[i] = (int64_t)slot3[3 * s + 2];
    }
}

// EXACT sharded path: receivers [s0, s1) of force/err (particle order) -> slot records
__global__ void k_pack_slot3(int64_t s0, int64_t s1, const double* __restrict__ force, const int64_t* __restrict__ err,
                             double* __restrict__ slot3) {
    for (int64_t i = s0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s1; i += (int64_t)gridDim.x * blockDim.x) {
        slot3[3 * i] = force[2 * i];
        slot3[3 * i + 1] = force[2 * i + 1];
        slot3[3 * i + 2] = (double)err[i];
    }
}

__global__ void k_unpack_slot3(int64_t n, const double* __restrict__ slot3, double* __restrict__ force,
                               int64_t* __restrict__ err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        force[2 * i] = slot3[3 * i];
        force[2 * i + 1] = slot3[3 * i + 1];
        err[i] = (int64_t)slot3[3 * i + 2];
    }
}

// exact re-scan (particle order) of receivers flagged -1: the reference's sentinel
__global__ void k_lr_rescan_pos(const double* __restrict__ pos, int64_t n, double L, double lo, double hi,
                                int64_t* __restrict__ err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (err[i] != -1) continue;
        const double xi = pos[2 * i], yi = pos[2 * i + 1];
        int64_t e = 0;
        for (int64_t k = 0; k < n; ++k) {
            if (k == i) continue;
            const double dx = mi_fast(xi - pos[2 * k], L, lo, hi), dy = mi_fast(yi - pos[2 * k + 1], L, lo, hi);
            if (dx * dx + dy * dy == 0.0) e = k + 1;
        }
        err[i] = e;
    }
}

#endif  // __CUDACC__

}  // namespace bd
