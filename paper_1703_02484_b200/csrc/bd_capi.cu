// bd_capi.cu -- extern "C" entry points of libbd_b200.so (include/bd_b200.h).
//
// Host side only launches: every loop of a step runs inside the persistent
// step kernels (bd_drivers.cuh, one source for the cooperative-grid and the
// single-CTA variants) or the all-pairs kernels (bd_allpairs*.cuh).  No
// entry point allocates device memory or synchronises the host.
#include <cuda_runtime.h>

#include <mutex>
#include <vector>

#include "bd_allpairs.cuh"
#include "bd_allpairs_sym.cuh"
#include "bd_drivers.cuh"
#include "bd_ops.cuh"
#include "bd_build.cuh"

using namespace bd;

namespace {

constexpr int STEP_BT = 256;
// The persistent step kernels exist twice: at <= 128 registers (2 CTAs per SM:
// fewer, cheaper grid barriers -- best while barrier latency dominates) and
// at 64 registers (4 CTAs per SM: twice the memory-level parallelism for the
// dependent gathers of large N; 25 % faster at N = 1M, 6 % at cfg3's 131k,
// slower at 16k and 65k: wide from N = 100k).
constexpr int WIDE_MINB = 4;
int64_t lrw_max_n() {  // BD_LRW_MAX_N overrides the EXACT warp-per-receiver threshold (tuning)
    static int64_t v = -1;
    if (v < 0) {
        const char* e = getenv("BD_LRW_MAX_N");
        v = e ? atoll(e) : LRW_MAX_N;
    }
    return v;
}

int64_t wide_min_n() {  // BD_WIDE_MIN_N overrides (tests: the two variants must agree bit for bit)
    static int64_t v = -1;
    if (v < 0) {
        const char* e = getenv("BD_WIDE_MIN_N");
        v = e ? atoll(e) : 100000;
    }
    return v;
}
constexpr int BLOCK_BT = 1024;

int g_num_sms = 0;
int g_grid_blocks_per_sm = 0;
int g_wide_blocks_per_sm = 0;
int g_lr_blocks_per_sm[2] = {1, 1};
int g_fast_blocks_per_sm = 1;
int g_smem_optin = 0;  // max dynamic shared memory per CTA (opt-in)
std::once_flag g_once;

int64_t block_max_n() {
    static int64_t v = -1;
    if (v < 0) {
        const char* e = getenv("BD_BLOCK_MAX_N");
        v = e ? atoll(e) : 768;  // one-CTA drivers up to here (B200: 0.129 vs 0.153 ms per O(N) step at 512, 0.192 vs 0.184 at 1,024)
    }
    return v;
}

BD_DEV Ctx make_ctx(const bd_state_t& s, const bd_params_t& p) {
    Ctx c;
    c.p = p;
    c.s = s;
    c.w = ws_carve(s.work, p, s.tri.ne, s.tri.nt);
    c.call = s.call ? *s.call : 0;
    ctx_init_work(c);
    return c;
}

// ---- persistent drivers: cooperative grid (barrier = grid.sync) and one CTA
// the triangulation step as one 1024-thread CTA per SM (big_min_n)
__global__ void __launch_bounds__(1024, 1) k_step_tri_grid_big(bd_state_t s, bd_params_t p, bd_stats_t* out) {
    Ctx c = make_ctx(s, p);
    ExecGrid x{c.w.ctl};
    step_tri_after_force(x, c, out);
}

template <int MINB>
__global__ void __launch_bounds__(STEP_BT, MINB) k_step_tri_grid(bd_state_t s, bd_params_t p, bd_stats_t* out) {
    Ctx c = make_ctx(s, p);
    ExecGrid x{c.w.ctl};
    step_tri_after_force(x, c, out);
}

// One-CTA drivers keep the control block's head (reduction ring, status,
// generation counters: everything before the grid-scan partials, which
// ExecBlock never uses) in shared memory for the launch: every phase ends in
// a reduction whose result all threads read right after the barrier, ~30
// cycles there instead of an L2 round trip.  Copied in at entry, out at exit.
constexpr int CTL_HEAD_WORDS = (int)(offsetof(Ctl, bsum) / sizeof(u64));

__device__ Ctl* ctl_in_smem(Ctl* g, u64* sm) {
    for (int k = threadIdx.x; k < CTL_HEAD_WORDS; k += blockDim.x) sm[k] = ((const u64*)g)[k];
    __syncthreads();
    return (Ctl*)sm;
}

__device__ void ctl_out_smem(Ctl* g, const u64* sm) {
    __syncthreads();
    for (int k = threadIdx.x; k < CTL_HEAD_WORDS; k += blockDim.x) ((u64*)g)[k] = sm[k];
}

__global__ void __launch_bounds__(BLOCK_BT) k_step_tri_block(bd_state_t s, bd_params_t p, bd_stats_t* out) {
    Ctx c = make_ctx(s, p);
    __shared__ u64 ctl_sm[CTL_HEAD_WORDS];
    Ctl* const ctl_g = c.w.ctl;
    c.w.ctl = ctl_in_smem(ctl_g, ctl_sm);
    ExecBlock x{c.w.ctl};
    step_tri_after_force(x, c, out);
    ctl_out_smem(ctl_g, ctl_sm);
}

// Small systems: the single-CTA driver keeps the triangulation, the
// positions and the per-step scratch it gathers through (incidence lists,
// flags, crossings) in shared memory for the whole step -- every phase is a
// chain of dependent gathers and atomics, ~30 cycles each there instead of
// ~600 from L2.  ~184 bytes per particle: N <= ~1200 within the 227 KB opt-in.
struct SmemState {
    int64_t tri_v, tri_shift, tri_edge, edge_v, edge_tri, edge_opp, pos, prev;
    int64_t inc_off, inc_cur, inc, eovl, estat, ewin, cross8, tinv, total;
};

BD_HD int64_t al16(int64_t x) { return (x + 15) & ~(int64_t)15; }

BD_HD SmemState smem_state(int64_t n, int64_t ne, int64_t nt) {
    SmemState l;
    int64_t o = 0;
    l.tri_v = o; o = al16(o + 12 * nt);
    l.tri_shift = o; o = al16(o + 6 * nt);
    l.tri_edge = o; o = al16(o + 12 * nt);
    l.edge_v = o; o = al16(o + 8 * ne);
    l.edge_tri = o; o = al16(o + 8 * ne);
    l.edge_opp = o; o = al16(o + 2 * ne);
    l.pos = o; o = al16(o + 16 * n);
    l.prev = o; o = al16(o + 16 * n);
    l.inc_off = o; o = al16(o + 4 * (n + 1));
    l.inc_cur = o; o = al16(o + 4 * n);
    l.inc = o; o = al16(o + 8 * ne);
    l.eovl = o; o = al16(o + ne);
    l.estat = o; o = al16(o + ne);
    l.ewin = o; o = al16(o + 4 * ne);
    l.cross8 = o; o = al16(o + 2 * n);
    l.tinv = o; o = al16(o + nt);
    l.total = o;
    return l;
}

__device__ void blk_copy(void* dst, const void* src, int64_t bytes) {
    int64_t done = 0;
    if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {  // 16 bytes per thread and step
        const int64_t v = bytes >> 4;
        for (int64_t i = threadIdx.x; i < v; i += blockDim.x) ((uint4*)dst)[i] = ((const uint4*)src)[i];
        done = v << 4;
    }
    for (int64_t i = done + threadIdx.x; i < bytes; i += blockDim.x) ((uint8_t*)dst)[i] = ((const uint8_t*)src)[i];
}

__global__ void __launch_bounds__(BLOCK_BT) k_step_tri_block_smem(bd_state_t s, bd_params_t p, bd_stats_t* out) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int64_t n = p.n, ne = s.tri.ne, nt = s.tri.nt;
    const SmemState l = smem_state(n, ne, nt);
    bd_state_t ls = s;
    ls.tri.tri_v = (int32_t*)(sm + l.tri_v);
    ls.tri.tri_shift = (int8_t*)(sm + l.tri_shift);
    ls.tri.tri_edge = (int32_t*)(sm + l.tri_edge);
    ls.tri.edge_v = (int32_t*)(sm + l.edge_v);
    ls.tri.edge_tri = (int32_t*)(sm + l.edge_tri);
    ls.tri.edge_opp = (int8_t*)(sm + l.edge_opp);
    ls.pos = (double*)(sm + l.pos);
    ls.prev = (double*)(sm + l.prev);
    blk_copy(ls.tri.tri_v, s.tri.tri_v, 12 * nt);
    blk_copy(ls.tri.tri_shift, s.tri.tri_shift, 6 * nt);
    blk_copy(ls.tri.tri_edge, s.tri.tri_edge, 12 * nt);
    blk_copy(ls.tri.edge_v, s.tri.edge_v, 8 * ne);
    blk_copy(ls.tri.edge_tri, s.tri.edge_tri, 8 * ne);
    blk_copy(ls.tri.edge_opp, s.tri.edge_opp, 2 * ne);
    blk_copy(ls.pos, s.pos, 16 * n);
    blk_copy(ls.prev, s.prev, 16 * n);
    for (int64_t i = threadIdx.x; i < ne; i += blockDim.x) ((uint32_t*)(sm + l.ewin))[i] = 0u;
    __syncthreads();
    Ctx c = make_ctx(ls, p);
    c.w.inc_off = (int32_t*)(sm + l.inc_off);  // scratch: rebuilt / rewritten before every use
    c.w.inc_cur = (int32_t*)(sm + l.inc_cur);
    c.w.inc = (int32_t*)(sm + l.inc);
    c.w.eovl = (uint8_t*)(sm + l.eovl);
    c.w.estat = (uint8_t*)(sm + l.estat);
    c.w.ewin = (uint32_t*)(sm + l.ewin);  // stamps: zeroed below (a stale shared-memory value could look current)
    c.w.cross8 = (int8_t*)(sm + l.cross8);
    c.w.tinv = (uint8_t*)(sm + l.tinv);
    __shared__ u64 ctl_sm[CTL_HEAD_WORDS];
    Ctl* const ctl_g = c.w.ctl;
    c.w.ctl = ctl_in_smem(ctl_g, ctl_sm);
    ExecBlock x{c.w.ctl};
    step_tri_after_force(x, c, out);
    ctl_out_smem(ctl_g, ctl_sm);
    __syncthreads();
    blk_copy(s.tri.tri_v, ls.tri.tri_v, 12 * nt);
    blk_copy(s.tri.tri_shift, ls.tri.tri_shift, 6 * nt);
    blk_copy(s.tri.tri_edge, ls.tri.tri_edge, 12 * nt);
    blk_copy(s.tri.edge_v, ls.tri.edge_v, 8 * ne);
    blk_copy(s.tri.edge_tri, ls.tri.edge_tri, 8 * ne);
    blk_copy(s.tri.edge_opp, ls.tri.edge_opp, 2 * ne);
    blk_copy(s.pos, ls.pos, 16 * n);
    blk_copy(s.prev, ls.prev, 16 * n);
}

template <int MINB>
__global__ void __launch_bounds__(STEP_BT, MINB) k_step_verlet_grid(bd_state_t s, bd_params_t p, bd_stats_t* out) {
    Ctx c = make_ctx(s, p);
    ExecGrid x{c.w.ctl};
    step_verlet(x, c, out);
}

__global__ void __launch_bounds__(BLOCK_BT) k_step_verlet_block(bd_state_t s, bd_params_t p, bd_stats_t* out) {
    Ctx c = make_ctx(s, p);
    __shared__ u64 ctl_sm[CTL_HEAD_WORDS];
    Ctl* const ctl_g = c.w.ctl;
    c.w.ctl = ctl_in_smem(ctl_g, ctl_sm);
    ExecBlock x{c.w.ctl};
    step_verlet(x, c, out);
    ctl_out_smem(ctl_g, ctl_sm);
}

template <int MINB>
__global__ void __launch_bounds__(STEP_BT, MINB) k_step_abp_grid(bd_state_t s, bd_params_t p, bd_stats_t* out) {
    Ctx c = make_ctx(s, p);
    ExecGrid x{c.w.ctl};
    step_abp(x, c, out);
}

__global__ void __launch_bounds__(BLOCK_BT) k_step_abp_block(bd_state_t s, bd_params_t p, bd_stats_t* out) {
    Ctx c = make_ctx(s, p);
    __shared__ u64 ctl_sm[CTL_HEAD_WORDS];
    Ctl* const ctl_g = c.w.ctl;
    c.w.ctl = ctl_in_smem(ctl_g, ctl_sm);
    ExecBlock x{c.w.ctl};
    step_abp(x, c, out);
    ctl_out_smem(ctl_g, ctl_sm);
}

template <class X>
__device__ void restore_delaunay_entry(X& x, Ctx& c, int64_t* passes_out) {
    Red<X> R(x);
    if (x.leader())
        for (int k = 0; k < 8; ++k) c.w.ctl->red[k] = 0;
    x.sync();
    const int64_t passes = restore_delaunay(x, R, c, 1000);
    if (x.leader()) passes_out[0] = passes;
}

__global__ void __launch_bounds__(STEP_BT) k_restore_delaunay_grid(bd_state_t s, bd_params_t p, int64_t* out) {
    Ctx c = make_ctx(s, p);
    ExecGrid x{c.w.ctl};
    restore_delaunay_entry(x, c, out);
}

// ---- method-boundary ops (bd_ops.cuh), one cooperative launch each --------
enum : int64_t {
    OP_INTEGRATE = 1, OP_APPLY_CROSSINGS, OP_EDGE_INVERSION, OP_SIGNED_AREA2, OP_DELAUNAY_FLAGS,
    OP_INVERTED_FLAGS, OP_FLIP_EDGES, OP_REPAIR, OP_RESTORE, OP_CORRECT_OVERLAPS, OP_INTEGRATE_NOISE
};

struct OpArgs {
    int64_t op, i0, i1;
    double d0;
    const void* in;
    void* out;
    int64_t* res;
};

__global__ void __launch_bounds__(STEP_BT) k_op_grid(bd_state_t s, bd_params_t p, OpArgs a) {
    Ctx c = make_ctx(s, p);
    ExecGrid x{c.w.ctl};
    switch (a.op) {
        case OP_INTEGRATE: op_integrate(x, c, a.d0, (int64_t*)a.out, a.res); break;
        case OP_APPLY_CROSSINGS: op_apply_crossings(x, c, (const int64_t*)a.in); break;
        case OP_EDGE_INVERSION: op_edge_inversion(x, c, a.res); break;
        case OP_SIGNED_AREA2: op_signed_area2(x, c, (double*)a.out); break;
        case OP_DELAUNAY_FLAGS: op_edge_flags(x, c, false, (uint8_t*)a.out); break;
        case OP_INVERTED_FLAGS: op_edge_flags(x, c, true, (uint8_t*)a.out); break;
        case OP_FLIP_EDGES: op_flip_edges(x, c, (const int64_t*)a.in, a.i0, a.res); break;
        case OP_REPAIR: op_repair_inversions(x, c, a.i0, a.i1 != 0, a.res); break;
        case OP_RESTORE: op_restore_delaunay(x, c, a.i0, a.res); break;
        case OP_CORRECT_OVERLAPS: op_correct_overlaps(x, c, a.i0, a.i1 != 0, a.res); break;
        case OP_INTEGRATE_NOISE: op_integrate(x, c, a.d0, (int64_t*)a.out, a.res, (const double*)a.in); break;
        default: break;
    }
}

// save_state / restore_state (triangulation.py:158-164)
__global__ void k_tri_copy(bd_tri_t a, bd_tri_t b) {
    struct Flat {
        BD_DEV int64_t tid() const { return blockIdx.x * (int64_t)blockDim.x + threadIdx.x; }
        BD_DEV int64_t nth() const { return (int64_t)gridDim.x * blockDim.x; }
    } x;
    ph_tri_copy(x, a, b);
}

// ---- kernel-boundary drop-ins over pair lists (cooperative grid) ----------

// build_cell_grid + cell_pairs (+ snapshot) into pair_a/pair_b; count[0]
__global__ void __launch_bounds__(STEP_BT) k_verlet_build_grid(bd_state_t s, bd_params_t p, int64_t* count) {
    Ctx c = make_ctx(s, p);
    ExecGrid x{c.w.ctl};
    Red<ExecGrid> R(x);
    if (x.leader()) {
        for (int k = 0; k < 8; ++k) c.w.ctl->red[k] = 0;
        c.w.ctl->status = 0;
        c.s.vl_meta[1] = 0;
    }
    x.sync();
    const bool ok = vl_rebuild(x, R, c, 0.0);
    if (x.leader()) count[0] = ok ? c.s.vl_meta[0] : (int64_t)c.w.ctl->err_i;
}

// short_range_kernel over a given pair list
__global__ void __launch_bounds__(STEP_BT) k_short_range_grid(bd_state_t s, bd_params_t p, int64_t npairs,
                                                              double* out, int64_t* err) {
    Ctx c = make_ctx(s, p);
    ExecGrid x{c.w.ctl};
    const ListPairs lp{c.s.pair_a, c.s.pair_b, npairs};
    build_incidence(x, p.n, lp, c.w.vinc_off, c.w.vinc_cur, c.w.vinc);
    sr_forces(x, c, out, err);
}

// overlap_pass_kernel over a given pair list: disp / flags / count (not applied)
__global__ void __launch_bounds__(STEP_BT) k_overlap_pass_grid(bd_state_t s, bd_params_t p, int64_t npairs,
                                                               double resolve, double* disp, uint8_t* flags,
                                                               int64_t* count) {
    Ctx c = make_ctx(s, p);
    ExecGrid x{c.w.ctl};
    Red<ExecGrid> R(x);
    if (x.leader())
        for (int k = 0; k < 8; ++k) c.w.ctl->red[k] = 0;
    x.sync();
    const ListPairs lp{c.s.pair_a, c.s.pair_b, npairs};
    build_incidence(x, p.n, lp, c.w.inc_off, c.w.inc_cur, c.w.inc);
    const double sigma = p.sigma, thresh = sigma * resolve;
    const double* pos = c.s.pos;
    u64* r = R.open();
    for (int64_t e = x.tid(); e < npairs; e += x.nth()) {
        const int64_t a = lp.a(e), b = lp.b(e);
        const double dx = mi_exact(pos[2 * b] - pos[2 * a], p), dy = mi_exact(pos[2 * b + 1] - pos[2 * a + 1], p);
        const double rr = sqrt(dx * dx + dy * dy);
        const bool ov = !(rr >= thresh || rr == 0.0);
        if (ov) {
            const double delta = sigma - rr;
            c.w.contrib[2 * e] = delta * (dx / rr);
            c.w.contrib[2 * e + 1] = delta * (dy / rr);
        }
        c.w.eovl[e] = (uint8_t)ov;
        R.add((u64)ov);
    }
    const u64 cnt = R.close(r);
    for (int64_t i = x.tid(); i < p.n; i += x.nth()) {
        double dx = 0.0, dy = 0.0;
        bool hit = false;
        for (int32_t j = c.w.inc_off[i]; j < c.w.inc_off[i + 1]; ++j) {
            const int64_t e = c.w.inc[j];
            if (!c.w.eovl[e]) continue;
            hit = true;
            if (lp.a(e) == i) {
                dx -= c.w.contrib[2 * e];
                dy -= c.w.contrib[2 * e + 1];
            } else {
                dx += c.w.contrib[2 * e];
                dy += c.w.contrib[2 * e + 1];
            }
        }
        disp[2 * i] = dx;
        disp[2 * i + 1] = dy;
        flags[i] = hit;
    }
    if (x.leader()) count[0] = (int64_t)cnt;
}

__global__ void k_max_sq_disp(const double* pos, const double* snap, int64_t n, bd_params_t p, unsigned long long* out) {
    unsigned long long best = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double dx = mi_exact(pos[2 * i] - snap[2 * i], p), dy = mi_exact(pos[2 * i + 1] - snap[2 * i + 1], p);
        const unsigned long long b = (unsigned long long)__double_as_longlong(dx * dx + dy * dy);
        best = b > best ? b : best;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, best, o);
        best = v > best ? v : best;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

// brute_force_overlaps (_kernels.py:239-275): every pair a < b with
// |mi(pos_b - pos_a)|^2 < thresh^2; count and the lexicographically first pair
__global__ void k_brute_overlaps(const double* pos, int64_t n, bd_params_t p, double thresh,
                                 unsigned long long* out) {
    const double t2 = thresh * thresh;
    unsigned long long cnt = 0, first = ~0ull;
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x) {
        for (int64_t b = a + 1; b < n; ++b) {
            const double dx = mi_exact(pos[2 * b] - pos[2 * a], p), dy = mi_exact(pos[2 * b + 1] - pos[2 * a + 1], p);
            if (dx * dx + dy * dy < t2) {
                ++cnt;
                const unsigned long long key = ((unsigned long long)a << 32) | (unsigned long long)b;
                first = key < first ? key : first;
            }
        }
    }
    if (cnt) {
        atomicAdd(&out[0], cnt);
        atomicMin(&out[1], first);
    }
}

__global__ void k_normals(uint64_t seed, uint64_t stream_id, uint64_t call, uint64_t purpose, int64_t npairs,
                          double* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npairs; i += (int64_t)gridDim.x * blockDim.x) {
        double z0, z1;
        normal_pair(seed, stream_id, call, (uint64_t)i, purpose, z0, z1);
        out[2 * i] = z0;
        out[2 * i + 1] = z1;
    }
}

__global__ void __launch_bounds__(STEP_BT) k_tri_build_grid(const double* pos, int64_t n, double L, bd_tri_t out,
                                                            void* work, int64_t* res) {
    BuildCtx c;
    c.g = build_geo(n, L);
    c.w = build_carve(work, n, L);
    c.pos = pos;
    c.out = out;
    ExecGrid x{c.w.ctl};
    Poly P, Q;
    tri_build(x, c, P, Q, res);
}

__global__ void k_audit_geometry(bd_tri_t T, const double* pos, double L, double tol, unsigned long long* out) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    unsigned long long bad_area = 0, bad_circ = 0;
    for (int64_t t = tid; t < T.nt; t += nth) {
        V2 xy[3];
        tri_xy(T, pos, L, t, xy);
        const double e1x = xy[1].x - xy[0].x, e1y = xy[1].y - xy[0].y;
        const double e2x = xy[2].x - xy[0].x, e2y = xy[2].y - xy[0].y;
        bad_area += (e1x * e2y - e1y * e2x <= 0.0);
    }
    for (int64_t e = tid; e < T.ne; e += nth) {
        V2 q[4];
        edge_quad(T, pos, L, e, q);
        bad_circ += incircle(q[0], q[1], q[2], q[3], tol);
    }
    if (bad_area) atomicAdd(&out[0], bad_area);
    if (bad_circ) atomicAdd(&out[1], bad_circ);
}

__global__ void k_probe_fp64(int64_t iters, double* out) {
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = 1e-9 * (double)(tid + j);
    const double m = 0.9999999, c = 1e-9;
    for (int64_t i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fma(a[j], m, c);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    out[tid & ((1 << 20) - 1)] = s;
}

int occupancy(const void* f, int bt) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, bt, 0);
    return nb > 0 ? nb : 1;
}

void init_device_info() {
    std::call_once(g_once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (const char* e = getenv("BD_WORKLIST_MIN_EDGES")) {
            const int64_t v = atoll(e);
            cudaMemcpyToSymbol(d_wl_min_edges, &v, sizeof(v));
        }
        int m = occupancy((const void*)k_step_tri_grid<2>, STEP_BT);
        const void* coop[] = {(const void*)k_restore_delaunay_grid, (const void*)k_op_grid, (const void*)k_tri_build_grid, (const void*)k_step_abp_grid<2>, (const void*)k_step_verlet_grid<2>,
                              (const void*)k_verlet_build_grid, (const void*)k_short_range_grid,
                              (const void*)k_overlap_pass_grid};
        for (const void* f : coop) {
            const int o = occupancy(f, STEP_BT);
            m = o < m ? o : m;
        }
        g_grid_blocks_per_sm = m;
        int mw = occupancy((const void*)k_step_tri_grid<WIDE_MINB>, STEP_BT);
        const void* wide[] = {(const void*)k_step_verlet_grid<WIDE_MINB>, (const void*)k_step_abp_grid<WIDE_MINB>};
        for (const void* f : wide) {
            const int o = occupancy(f, STEP_BT);
            mw = o < mw ? o : mw;
        }
        g_wide_blocks_per_sm = mw;
        g_lr_blocks_per_sm[1] = occupancy((const void*)k_allpairs<true>, LR_BT);
        g_lr_blocks_per_sm[0] = occupancy((const void*)k_allpairs<false>, LR_BT);
        g_fast_blocks_per_sm = occupancy((const void*)k_allpairs_fast, FS_BT);
        cudaFuncSetAttribute((const void*)k_allpairs_sym, cudaFuncAttributeMaxDynamicSharedMemorySize, SY_SMEM);
        cudaDeviceGetAttribute(&g_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        int st = 0;
        cudaFuncAttributes fa;
        if (cudaFuncGetAttributes(&fa, (const void*)k_step_tri_block_smem) == cudaSuccess) st = (int)fa.sharedSizeBytes;
        g_smem_optin -= st;
        cudaFuncSetAttribute((const void*)k_step_tri_block_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             g_smem_optin);
    });
}

int64_t grid_cap_per_sm() {  // BD_GRID_BLOCKS_PER_SM caps the persistent grids (tuning)
    static int64_t v = -1;
    if (v < 0) {
        const char* e = getenv("BD_GRID_BLOCKS_PER_SM");
        v = e ? atoll(e) : 0;
    }
    return v;
}

int grid_blocks(int64_t work_items, bool wide = false, int64_t per_sm_cap = 0) {
    int64_t want = (work_items + STEP_BT - 1) / STEP_BT;
    int64_t per = wide ? g_wide_blocks_per_sm : g_grid_blocks_per_sm;
    if (per_sm_cap > 0 && per_sm_cap < per) per = per_sm_cap;
    if (grid_cap_per_sm() > 0 && grid_cap_per_sm() < per) per = grid_cap_per_sm();
    int64_t cap = (int64_t)g_num_sms * per;
    if (cap > 4096) cap = 4096;
    if (want > cap) want = cap;
    return (int)(want < 1 ? 1 : want);
}

int err_code(cudaError_t e) { return e == cudaSuccess ? 0 : -(int)e; }

unsigned grid_for(int64_t items, int bt = 256) {
    int64_t nb = (items + bt - 1) / bt;
    if (nb > 8 * (int64_t)g_num_sms) nb = 8 * (int64_t)g_num_sms;
    return (unsigned)(nb < 1 ? 1 : nb);
}

int coop_launch(const void* f, int64_t items, void** args, cudaStream_t st, bool wide = false,
                int64_t per_sm_cap = 0) {
    return err_code(
        cudaLaunchCooperativeKernel(f, dim3(grid_blocks(items, wide, per_sm_cap)), dim3(STEP_BT), args, 0, st));
}

// Below this many particles the step drivers run one CTA per SM: the grid
// barriers (~100 per step) dominate and get cheaper with fewer CTAs
// (cfg2, N = 16k: 0.31 -> 0.25 ms per step); above it the phases' work
// dominates and two CTAs per SM win (cfg3: 0.81 vs 1.0 ms).
int64_t narrow_max_n() {  // BD_NARROW_MAX_N overrides (tests run both grid shapes on the goldens)
    static int64_t v = -1;
    if (v < 0) {
        const char* e = getenv("BD_NARROW_MAX_N");
        v = e ? atoll(e) : 65536;
    }
    return v;
}

// ---- all-pairs launches ------------------------------------------------------

// EXACT (and unsorted FAST for receiver sub-ranges): one wave of equally
// loaded CTAs, 148 x m CTAs, m the smallest multiple of SMs holding every
// receiver at <= LR_BT per CTA (more waves only past the residency limit)
int launch_lr(const double4* src, const double* mu, int64_t n, const bd_params_t& p, int64_t i0, int64_t i1,
              int precision, double* out, int64_t* err, cudaStream_t st) {
    if (i1 <= i0) return 0;
    const int fast = precision == BD_LR_FAST;
    const int64_t R = i1 - i0;
    if (!fast && n <= lrw_max_n()) {
        k_allpairs_exact_warp<<<(unsigned)((R + LRW_WARPS - 1) / LRW_WARPS), LRW_WARPS * 32, 0, st>>>(
            src, mu, n, p.L, p.mi_lo, p.mi_hi, i0, i1, out, err);
        return err_code(cudaGetLastError());
    }
    const int64_t nb_min = (R + LR_BT - 1) / LR_BT;
    const int64_t m = (nb_min + g_num_sms - 1) / g_num_sms;
    int64_t nb = m <= g_lr_blocks_per_sm[fast] ? (int64_t)g_num_sms * m : nb_min;
    if (nb > R) nb = R;
    const int64_t per_block = (R + nb - 1) / nb;
    nb = (R + per_block - 1) / per_block;
    if (fast) {
        k_allpairs<true><<<(unsigned)nb, LR_BT, 0, st>>>(src, mu, n, p.L, p.mi_lo, p.mi_hi, i0, i1, per_block, out,
                                                           err);
        k_lr_rescan<<<grid_for(R), 256, 0, st>>>(src, n, p.L, p.mi_lo, p.mi_hi, i0, i1, err);
    } else {
        k_allpairs<false><<<(unsigned)nb, LR_BT, 0, st>>>(src, mu, n, p.L, p.mi_lo, p.mi_hi, i0, i1, per_block, out,
                                                            err);
    }
    return err_code(cudaGetLastError());
}

int launch_pack(const double* pos, const double* alpha, int64_t n, double4* src, cudaStream_t st) {
    k_pack_sources<<<grid_for(n), 256, 0, st>>>(pos, alpha, n, src);
    return err_code(cudaGetLastError());
}

// FAST stage 1: Morton counting sort + 48-byte source packing + tile boxes
int launch_fast_prepare(const double* pos, const double* alpha, const double* mu, int64_t n, double L,
                        const SortWs& w, cudaStream_t st) {
    const int64_t nc = fast_ncells(n);
    cudaError_t e = cudaMemsetAsync(w.cell_off, 0, sizeof(int32_t) * (nc + 1), st);
    if (e != cudaSuccess) return err_code(e);
    k_sort_count<<<grid_for(n), 256, 0, st>>>(pos, n, L, w);
    k_sort_scan<<<1, 1024, 0, st>>>(w, nc);
    k_sort_scatter<<<grid_for(n), 256, 0, st>>>(n, w);
    k_sort_fix<<<grid_for(nc), 256, 0, st>>>(nc, w);
    k_pack6<<<(unsigned)((n + FS_TS - 1) / FS_TS), FS_TS, 0, st>>>(pos, alpha, mu, n, w);
    return err_code(cudaGetLastError());
}

// FAST stage 2: receivers = sorted slots [s0, s1)
int launch_fast_slots(int64_t n, const bd_params_t& p, int64_t s0, int64_t s1, const SortWs& w, double* slot3,
                      cudaStream_t st) {
    if (s1 <= s0) return 0;
    const int64_t nb = (s1 - s0 + FS_RPB - 1) / FS_RPB;
    k_allpairs_fast<<<dim3((unsigned)nb, (unsigned)w.splits), FS_BT, 0, st>>>(w, n, p.L, p.mi_lo, p.mi_hi, s0, s1,
                                                                               slot3);
    if (w.splits > 1) k_reduce_parts<<<grid_for(s1 - s0), 256, 0, st>>>(s0, s1, n, w, slot3);
    return err_code(cudaGetLastError());
}

// FAST stage 3: slots -> particle order; exact re-scan of flagged receivers
int launch_fast_finish(const double* pos, int64_t n, const bd_params_t& p, const SortWs& w, const double* slot3,
                       double* out, int64_t* err, cudaStream_t st) {
    k_unsort_forces<<<grid_for(n), 256, 0, st>>>(0, n, w, slot3, out, err);
    k_lr_rescan_pos<<<grid_for(n), 256, 0, st>>>(pos, n, p.L, p.mi_lo, p.mi_hi, err);
    return err_code(cudaGetLastError());
}

// FAST-SYM stage 1 (every rank): sort + pack; pair kernel over this rank's
// chunks; its partial P_r = A_r - B_r per slot into `part`
// ---- kernel timing ring (measurement): CUDA events recorded around each
// launch of the all-pairs pair kernel while enabled (bd_timing_enable), on the
// launching stream; bench.py reads the per-launch device times back for the
// roofline of the dominant kernel
struct TimingRing {
    std::vector<cudaEvent_t> ev;
    int64_t next = 0, cap = 0;
};
TimingRing g_tr;

void timing_begin(cudaStream_t st) {
    if (g_tr.cap && g_tr.next < g_tr.cap) cudaEventRecord(g_tr.ev[2 * g_tr.next], st);
}
void timing_end(cudaStream_t st) {
    if (g_tr.cap && g_tr.next < g_tr.cap) cudaEventRecord(g_tr.ev[2 * g_tr.next++ + 1], st);
}

int launch_sym_partial(const double* pos, const double* alpha, const double* mu, int64_t n, const bd_params_t& p,
                       const SymWs& w, int rank, int world, double* part, cudaStream_t st) {
    init_device_info();
    if (n <= 0) return 0;
    // (alpha group, Morton cell) with ~8 particles per cell: tiles of 256
    // slots stay as compact, and the single-CTA scan has 8x fewer cells
    SortWs sw = w.sort;
    sw.grid_log2 = sw.grid_log2 > 2 ? sw.grid_log2 - 1 : sw.grid_log2;
    const int64_t nc = 2 * ((int64_t)1 << (2 * sw.grid_log2));
    // receivers that can meet an image tie (EDGE mode only for those): coordinate buckets
    const int64_t nb = 2 * sym_tie_buckets(n);
    cudaError_t e = cudaMemsetAsync(sw.cell_off, 0, sizeof(int32_t) * (nc + 1), st);
    if (e != cudaSuccess) return err_code(e);
    e = cudaMemsetAsync(w.tcnt, 0, sizeof(int32_t) * (nb + 1), st);
    if (e != cudaSuccess) return err_code(e);
    // sort + tie buckets: one counting pass, both scans in one launch, one scatter pass
    k_sym_count<<<grid_for(n), 256, 0, st>>>(pos, alpha, n, p.L, sw, w);
    {
        SortWs tb = w.sort;
        tb.cell_off = w.tcnt;
        tb.cell_cur = w.tcur;
        k_sort_scan2<<<2, 1024, 0, st>>>(sw, nc, tb, nb);
    }
    k_sym_scatter<<<grid_for(n), 256, 0, st>>>(pos, n, p.L, sw, w);
    k_sort_fix<<<grid_for(nc), 256, 0, st>>>(nc, sw);
    k_sym_pack<<<(unsigned)sym_tiles(n), SY_TS, 0, st>>>(pos, alpha, mu, n, p.L, p.mi_lo, p.mi_hi, w);
    const SymRange g = sym_range(n, rank, world);
    const int nch = g.nch;
    if (nch > 0 || g.i1 > g.i0) {
        timing_begin(st);
        k_allpairs_sym<<<dim3((unsigned)sym_blocks(n), (unsigned)(1 + nch)), SY_CT, SY_SMEM, st>>>(
            w, n, p.L, p.mi_lo, p.mi_hi, g.c0, g.cs, g.i0, g.i1);
        timing_end(st);
    }
    k_sym_partial<<<grid_for(n), 256, 0, st>>>(n, w, g, part);
    return err_code(cudaGetLastError());
}

// FAST-SYM stage 2: F = mu P (P summed over the ranks), unsort, exact re-scan of flagged receivers
int launch_sym_finish(const double* pos, int64_t n, const bd_params_t& p, const SymWs& w, const double* part,
                      double* out, int64_t* err, cudaStream_t st) {
    if (n <= 0) return 0;
    k_sym_finish<<<grid_for(n), 256, 0, st>>>(n, w, part, out, err);
    k_lr_rescan_pos<<<grid_for(n), 256, 0, st>>>(pos, n, p.L, p.mi_lo, p.mi_hi, err);
    return err_code(cudaGetLastError());
}

// FAST-SYM on one GPU
int launch_sym(const double* pos, const double* alpha, const double* mu, int64_t n, const bd_params_t& p,
               const SymWs& w, double* out, int64_t* err, cudaStream_t st) {
    int rc = launch_sym_partial(pos, alpha, mu, n, p, w, 0, 1, w.part, st);
    if (rc) return rc;
    return launch_sym_finish(pos, n, p, w, w.part, out, err, st);
}

int launch_force(const bd_state_t* s, const bd_params_t* p, cudaStream_t st) {
    init_device_info();
    if (p->force_mode == BD_FORCE_SR) return 0;  // the short-range force runs inside the step kernel
    const Ws w = ws_carve(s->work, *p, s->tri.ne, s->tri.nt);
    // force on the pre-move positions (dynamics.py:194)
    if (p->lr_precision == BD_LR_FAST_SYM)
        return launch_sym(s->pos, s->alpha, s->mu, p->n, *p, sym_ws_carve(w.src4, p->n), s->force, s->force_err, st);
    if (p->lr_precision == BD_LR_FAST) {
        const SortWs fw = fast_ws_carve(w.src4, p->n);
        int rc = launch_fast_prepare(s->pos, s->alpha, s->mu, p->n, p->L, fw, st);
        if (rc) return rc;
        rc = launch_fast_slots(p->n, *p, 0, p->n, fw, fw.slot3, st);
        if (rc) return rc;
        return launch_fast_finish(s->pos, p->n, *p, fw, fw.slot3, s->force, s->force_err, st);
    }
    int rc = launch_pack(s->pos, s->alpha, p->n, (double4*)w.src4, st);
    if (rc) return rc;
    return launch_lr((const double4*)w.src4, s->mu, p->n, *p, 0, p->n, (int)p->lr_precision, s->force,
                     s->force_err, st);
}

// From this many particles the triangulation step runs as one 1024-thread CTA
// per SM (k_step_tri_grid_big) instead of 4 x 256: the same threads, a
// quarter of the barrier arrivals (grid.sync 1.27 vs 1.63 us): cfg3 O(N)
// step 0.69 -> 0.63 ms; from 32k since the per-CTA control-word reads
// (O(N) step at 16k / 32k / 48k / 64k: 0.277 vs 0.248, 0.351 vs 0.357,
// 0.378 vs 0.476, 0.577 vs 0.616 ms).  BD_BIG_MIN_N overrides (0: off).
int64_t big_min_n() {
    static int64_t v = -1;
    if (v < 0) {
        const char* e = getenv("BD_BIG_MIN_N");
        v = e ? atoll(e) : 32768;
    }
    return v;
}

int launch_driver(const void* grid_fn, const void* wide_fn, const void* block_fn, const bd_state_t* s,
                  const bd_params_t* p, bd_stats_t* out, cudaStream_t st) {
    init_device_info();
    bd_state_t sv = *s;
    bd_params_t pv = *p;
    void* args[] = {&sv, &pv, &out};
    if (big_min_n() > 0 && p->n >= big_min_n() && wide_fn == (const void*)k_step_tri_grid<WIDE_MINB>)
        return err_code(cudaLaunchCooperativeKernel((const void*)k_step_tri_grid_big, dim3(g_num_sms), dim3(1024),
                                                    args, 0, st));
    if (p->n <= block_max_n())
        return err_code(cudaLaunchKernel(block_fn, dim3(1), dim3(BLOCK_BT), args, 0, st));
    int64_t items = s->tri.ne > p->n ? s->tri.ne : p->n;
    if (p->pair_capacity > items) items = p->pair_capacity;
    if (p->n >= wide_min_n()) return coop_launch(wide_fn, items, args, st, true);
    return coop_launch(grid_fn, items, args, st, false, p->n < narrow_max_n() ? 1 : 0);
}

int64_t smem_driver_enabled() {  // BD_SMEM_DRIVER=0 turns the shared-memory single-CTA driver off
    static int64_t v = -1;
    if (v < 0) {
        const char* e = getenv("BD_SMEM_DRIVER");
        v = (e && atoi(e) == 0) ? 0 : 1;
    }
    return v;
}

int launch_maintain_tri(const bd_state_t* s, const bd_params_t* p, bd_stats_t* out, cudaStream_t st) {
    init_device_info();
    if (p->n <= block_max_n() && smem_driver_enabled()) {
        const int64_t bytes = smem_state(p->n, s->tri.ne, s->tri.nt).total;
        if (bytes <= g_smem_optin) {
            bd_state_t sv = *s;
            bd_params_t pv = *p;
            void* args[] = {&sv, &pv, &out};
            return err_code(cudaLaunchKernel((const void*)k_step_tri_block_smem, dim3(1), dim3(BLOCK_BT), args,
                                             (size_t)bytes, st));
        }
    }
    return launch_driver((const void*)k_step_tri_grid<2>, (const void*)k_step_tri_grid<WIDE_MINB>,
                         (const void*)k_step_tri_block, s, p, out, st);
}

int launch_step_tri(const bd_state_t* s, const bd_params_t* p, bd_stats_t* out, cudaStream_t st) {
    int rc = launch_force(s, p, st);
    if (rc) return rc;
    return launch_maintain_tri(s, p, out, st);
}

int launch_step_verlet(const bd_state_t* s, const bd_params_t* p, bd_stats_t* out, cudaStream_t st) {
    return launch_driver((const void*)k_step_verlet_grid<2>, (const void*)k_step_verlet_grid<WIDE_MINB>,
                         (const void*)k_step_verlet_block, s, p, out, st);
}

int launch_op(const bd_state_t* s, const bd_params_t* p, OpArgs a, int64_t items, cudaStream_t st) {
    init_device_info();
    bd_state_t sv = *s;
    bd_params_t pv = *p;
    void* args[] = {&sv, &pv, &a};
    if (items < p->n) items = p->n;
    return coop_launch((const void*)k_op_grid, items, args, st);
}

int launch_step_abp(const bd_state_t* s, const bd_params_t* p, bd_stats_t* out, cudaStream_t st) {
    return launch_driver((const void*)k_step_abp_grid<2>, (const void*)k_step_abp_grid<WIDE_MINB>,
                         (const void*)k_step_abp_block, s, p, out, st);
}

// a transient state for the standalone pair-list entry points
struct PairCtx {
    bd_params_t p;
    bd_state_t s;
    int64_t meta[4];
};

bool pair_ctx(PairCtx& pc, const double* pos, int64_t n, double L, double r_list, int64_t capacity, void* work) {
    memset(&pc, 0, sizeof(pc));
    pc.p.n = n;
    pc.p.L = L;
    pc.p.sigma = 1.0;
    pc.p.skin = 0.0;
    pc.p.r_cut = r_list;
    prepare_params(&pc.p);
    pc.p.r_list = r_list;
    const int64_t ncx = (int64_t)floor(L / r_list);
    pc.p.ncx = ncx < 3 ? 0 : ncx;
    pc.p.pair_capacity = capacity > 0 ? capacity : 1;
    const WsLayout l = ws_layout(pc.p, 0, 0);
    char* b = (char*)work;
    pc.s.pos = (double*)pos;
    pc.s.work = b;
    pc.s.work_bytes = l.total;
    pc.s.vl_snap = (double*)(b + l.total);
    pc.s.vl_meta = (int64_t*)(b + l.total + align_up(16 * n));
    return true;
}

int64_t pair_ws_bytes(int64_t n, double L, double r_list, int64_t n_pairs) {
    PairCtx pc;
    memset(&pc, 0, sizeof(pc));
    pc.p.n = n;
    pc.p.L = L;
    const int64_t ncx = r_list > 0 ? (int64_t)floor(L / r_list) : 0;
    pc.p.ncx = ncx < 3 ? 0 : ncx;
    pc.p.pair_capacity = n_pairs > 0 ? n_pairs : 1;
    return ws_layout(pc.p, 0, 0).total + align_up(16 * n) + 256;
}

}  // namespace

extern "C" {

void bd_prepare_params(bd_params_t* p) { prepare_params(p); }

int64_t bd_workspace_bytes(const bd_params_t* p, int64_t ne, int64_t nt) { return ws_layout(*p, ne, nt).total; }

int64_t bd_pairs_workspace_bytes(int64_t n, double L, double r_list, int64_t n_pairs) {
    return pair_ws_bytes(n, L, r_list, n_pairs);
}

int64_t bd_long_range_workspace_bytes(int64_t n) {
    const int64_t f = fast_ws_bytes(n);
    return (f > 32 * n ? f : 32 * n) + 512;
}

int64_t bd_long_range_workspace_bytes_for(int64_t n, int precision) {
    if (precision == BD_LR_FAST_SYM) return sym_ws_bytes(n) + 512;
    return bd_long_range_workspace_bytes(n);
}

int bd_long_range_forces(const double* pos, const double* alpha, const double* mu, int64_t n, double L, int64_t i_begin,
                         int64_t i_end, int precision, double* out, int64_t* err, void* work, void* stream) {
    init_device_info();
    cudaStream_t st = (cudaStream_t)stream;
    bd_params_t p;
    memset(&p, 0, sizeof(p));
    p.L = L;
    prepare_params(&p);
    if (precision == BD_LR_FAST_SYM) {
        if (i_begin != 0 || i_end != n) return -(int)cudaErrorInvalidValue;  // whole range only
        return launch_sym(pos, alpha, mu, n, p, sym_ws_carve(work, n), out, err, st);
    }
    if (precision == BD_LR_FAST && i_begin == 0 && i_end == n) {
        const SortWs fw = fast_ws_carve(work, n);
        int rc = launch_fast_prepare(pos, alpha, mu, n, L, fw, st);
        if (rc) return rc;
        rc = launch_fast_slots(n, p, 0, n, fw, fw.slot3, st);
        if (rc) return rc;
        return launch_fast_finish(pos, n, p, fw, fw.slot3, out, err, st);
    }
    int rc = launch_pack(pos, alpha, n, (double4*)work, st);
    if (rc) return rc;
    return launch_lr((const double4*)work, mu, n, p, i_begin, i_end, precision, out, err, st);
}

int bd_verlet_build(const double* pos, int64_t n, double L, double r_list, int64_t* pair_a, int64_t* pair_b,
                    int64_t capacity, int64_t* count, void* work, void* stream) {
    init_device_info();
    PairCtx pc;
    pair_ctx(pc, pos, n, L, r_list, capacity, work);
    pc.s.pair_a = pair_a;
    pc.s.pair_b = pair_b;
    void* args[] = {&pc.s, &pc.p, &count};
    return coop_launch((const void*)k_verlet_build_grid, n > capacity ? n : capacity, args, (cudaStream_t)stream);
}

int bd_short_range_forces(const double* pos, const double* alpha, const double* mu, int64_t n, const int64_t* pair_a,
                          const int64_t* pair_b, int64_t n_pairs, double L, double r_cut, double* out, int64_t* err,
                          void* work, void* stream) {
    init_device_info();
    PairCtx pc;
    pair_ctx(pc, pos, n, L, 0.0, n_pairs, work);
    pc.p.ncx = 0;
    pc.p.r_cut = r_cut;
    pc.s.alpha = (double*)alpha;
    pc.s.mu = (double*)mu;
    pc.s.pair_a = (int64_t*)pair_a;
    pc.s.pair_b = (int64_t*)pair_b;
    void* args[] = {&pc.s, &pc.p, &n_pairs, &out, &err};
    return coop_launch((const void*)k_short_range_grid, n > n_pairs ? n : n_pairs, args, (cudaStream_t)stream);
}

int bd_overlap_pass(const double* pos, int64_t n, const int64_t* pair_a, const int64_t* pair_b, int64_t n_pairs,
                    double L, double sigma, double resolve, double* disp, uint8_t* flags, int64_t* count, void* work,
                    void* stream) {
    init_device_info();
    PairCtx pc;
    pair_ctx(pc, pos, n, L, 0.0, n_pairs, work);
    pc.p.ncx = 0;
    pc.p.sigma = sigma;
    pc.s.pair_a = (int64_t*)pair_a;
    pc.s.pair_b = (int64_t*)pair_b;
    void* args[] = {&pc.s, &pc.p, &n_pairs, &resolve, &disp, &flags, &count};
    return coop_launch((const void*)k_overlap_pass_grid, n > n_pairs ? n : n_pairs, args, (cudaStream_t)stream);
}

int bd_max_sq_displacement(const double* pos, const double* snap, int64_t n, double L, double* out, void* stream) {
    init_device_info();
    bd_params_t p;
    memset(&p, 0, sizeof(p));
    p.L = L;
    prepare_params(&p);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), st);
    if (e != cudaSuccess) return err_code(e);
    k_max_sq_disp<<<grid_for(n), 256, 0, st>>>(pos, snap, n, p, (unsigned long long*)out);
    return err_code(cudaGetLastError());
}

int bd_brute_overlaps(const double* pos, int64_t n, double L, double thresh, int64_t* out, void* stream) {
    init_device_info();
    bd_params_t p;
    memset(&p, 0, sizeof(p));
    p.L = L;
    prepare_params(&p);
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned long long init[2] = {0ull, ~0ull};
    cudaError_t e = cudaMemcpyAsync(out, init, sizeof(init), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return err_code(e);
    k_brute_overlaps<<<grid_for(n, 128), 128, 0, st>>>(pos, n, p, thresh, (unsigned long long*)out);
    return err_code(cudaGetLastError());
}

int bd_normals(uint64_t seed, uint64_t stream_id, uint64_t call, uint64_t purpose, int64_t n_pairs, double* out,
               void* stream) {
    init_device_info();
    k_normals<<<grid_for(n_pairs), 256, 0, (cudaStream_t)stream>>>(seed, stream_id, call, purpose, n_pairs, out);
    return err_code(cudaGetLastError());
}

int bd_force(const bd_state_t* s, const bd_params_t* p, void* stream) {
    return launch_force(s, p, (cudaStream_t)stream);
}

// ---- sharded all-pairs force (multi-GPU: receiver slots per rank + all-gather)
int bd_force_sym_partial(const bd_state_t* s, const bd_params_t* p, int rank, int world, double* part,
                         void* stream) {
    if (p->lr_precision != BD_LR_FAST_SYM || world < 1 || rank < 0 || rank >= world)
        return -(int)cudaErrorInvalidValue;
    const Ws w = ws_carve(s->work, *p, s->tri.ne, s->tri.nt);
    return launch_sym_partial(s->pos, s->alpha, s->mu, p->n, *p, sym_ws_carve(w.src4, p->n), rank, world, part,
                              (cudaStream_t)stream);
}

int bd_sym_shard(int64_t n, int rank, int world, int64_t* out) {
    if (n < 0 || world < 1 || rank < 0 || rank >= world || !out) return -(int)cudaErrorInvalidValue;
    const SymRange g = sym_range(n, rank, world);
    const int64_t D = sym_D(n);
    const int64_t v[11] = {SY_BT, sym_blocks(n), D, sym_chunks(n), sym_per(n), g.c0, g.cs, g.nch, 0,
                           g.i0, g.i1};
    for (int k = 0; k < 11; ++k) out[k] = v[k];
    return 0;
}

int bd_force_sym_finish(const bd_state_t* s, const bd_params_t* p, const double* part, void* stream) {
    if (p->lr_precision != BD_LR_FAST_SYM) return -(int)cudaErrorInvalidValue;
    const Ws w = ws_carve(s->work, *p, s->tri.ne, s->tri.nt);
    return launch_sym_finish(s->pos, p->n, *p, sym_ws_carve(w.src4, p->n), part, s->force, s->force_err,
                             (cudaStream_t)stream);
}

int bd_force_prepare(const bd_state_t* s, const bd_params_t* p, void* stream) {
    init_device_info();
    if (p->lr_precision == BD_LR_FAST_SYM) return -(int)cudaErrorInvalidValue;  // bd_force_sym_partial
    cudaStream_t st = (cudaStream_t)stream;
    if (p->force_mode == BD_FORCE_SR) return 0;
    const Ws w = ws_carve(s->work, *p, s->tri.ne, s->tri.nt);
    if (p->lr_precision == BD_LR_FAST)
        return launch_fast_prepare(s->pos, s->alpha, s->mu, p->n, p->L, fast_ws_carve(w.src4, p->n), st);
    return launch_pack(s->pos, s->alpha, p->n, (double4*)w.src4, st);
}

int bd_force_slots(const bd_state_t* s, const bd_params_t* p, int64_t s0, int64_t s1, double* slot3, void* stream) {
    init_device_info();
    cudaStream_t st = (cudaStream_t)stream;
    if (p->force_mode == BD_FORCE_SR) return 0;
    if (s1 > p->n) s1 = p->n;
    if (s1 <= s0) return 0;
    const Ws w = ws_carve(s->work, *p, s->tri.ne, s->tri.nt);
    if (p->lr_precision == BD_LR_FAST)
        return launch_fast_slots(p->n, *p, s0, s1, fast_ws_carve(w.src4, p->n), slot3, st);
    int rc = launch_lr((const double4*)w.src4, s->mu, p->n, *p, s0, s1, BD_LR_EXACT, s->force, s->force_err, st);
    if (rc) return rc;
    k_pack_slot3<<<grid_for(s1 - s0), 256, 0, st>>>(s0, s1, s->force, s->force_err, slot3);
    return err_code(cudaGetLastError());
}

int bd_force_finish(const bd_state_t* s, const bd_params_t* p, const double* slot3, void* stream) {
    init_device_info();
    cudaStream_t st = (cudaStream_t)stream;
    if (p->force_mode == BD_FORCE_SR) return 0;
    const Ws w = ws_carve(s->work, *p, s->tri.ne, s->tri.nt);
    if (p->lr_precision == BD_LR_FAST)
        return launch_fast_finish(s->pos, p->n, *p, fast_ws_carve(w.src4, p->n), slot3, s->force, s->force_err, st);
    k_unpack_slot3<<<grid_for(p->n), 256, 0, st>>>(p->n, slot3, s->force, s->force_err);
    return err_code(cudaGetLastError());
}

int bd_maintain_tri(const bd_state_t* s, const bd_params_t* p, bd_stats_t* out, void* stream) {
    return launch_maintain_tri(s, p, out, (cudaStream_t)stream);
}

int bd_step_tri(const bd_state_t* s, const bd_params_t* p, void* stream) {
    return launch_step_tri(s, p, s->stats, (cudaStream_t)stream);
}

int bd_run_tri(const bd_state_t* s, const bd_params_t* p, int64_t steps, bd_stats_t* stats_out, void* stream) {
    for (int64_t j = 0; j < steps; ++j) {
        int rc = launch_step_tri(s, p, stats_out + j, (cudaStream_t)stream);
        if (rc) return rc;
    }
    return 0;
}

int bd_step_verlet(const bd_state_t* s, const bd_params_t* p, bd_stats_t* stats_out, void* stream) {
    return launch_step_verlet(s, p, stats_out, (cudaStream_t)stream);
}

int bd_run_verlet(const bd_state_t* s, const bd_params_t* p, int64_t steps, bd_stats_t* stats_out, void* stream) {
    for (int64_t j = 0; j < steps; ++j) {
        int rc = launch_step_verlet(s, p, stats_out + j, (cudaStream_t)stream);
        if (rc) return rc;
    }
    return 0;
}

int bd_step_abp(const bd_state_t* s, const bd_params_t* p, bd_stats_t* stats_out, void* stream) {
    return launch_step_abp(s, p, stats_out, (cudaStream_t)stream);
}

int bd_run_abp(const bd_state_t* s, const bd_params_t* p, int64_t steps, bd_stats_t* stats_out, void* stream) {
    for (int64_t j = 0; j < steps; ++j) {
        int rc = launch_step_abp(s, p, stats_out + j, (cudaStream_t)stream);
        if (rc) return rc;
    }
    return 0;
}

int bd_clear_status(const bd_state_t* s, void* stream) {
    Ctl* ctl = (Ctl*)s->work;  // the control block heads every workspace
    return err_code(cudaMemsetAsync(&ctl->status, 0, 3 * sizeof(unsigned long long), (cudaStream_t)stream));
}

int bd_tri_restore_delaunay(const bd_state_t* s, const bd_params_t* p, int64_t* passes_out, void* stream) {
    init_device_info();
    bd_state_t sv = *s;
    bd_params_t pv = *p;
    void* args[] = {&sv, &pv, &passes_out};
    const int64_t items = s->tri.ne > p->n ? s->tri.ne : p->n;
    return coop_launch((const void*)k_restore_delaunay_grid, items, args, (cudaStream_t)stream);
}

int bd_integrate(const bd_state_t* s, const bd_params_t* p, double dt, int64_t* crossings, int64_t* result,
                 void* stream) {
    return launch_op(s, p, OpArgs{OP_INTEGRATE, 0, 0, dt, nullptr, crossings, result}, p->n, (cudaStream_t)stream);
}

int bd_integrate_noise(const bd_state_t* s, const bd_params_t* p, double dt, const double* noise, int64_t* crossings,
                       int64_t* result, void* stream) {
    if (!noise) return -(int)cudaErrorInvalidValue;
    return launch_op(s, p, OpArgs{OP_INTEGRATE_NOISE, 0, 0, dt, noise, crossings, result}, p->n,
                     (cudaStream_t)stream);
}

int bd_tri_apply_crossings(const bd_state_t* s, const bd_params_t* p, const int64_t* crossings, void* stream) {
    return launch_op(s, p, OpArgs{OP_APPLY_CROSSINGS, 0, 0, 0.0, crossings, nullptr, nullptr}, s->tri.nt,
                     (cudaStream_t)stream);
}

int bd_tri_edge_inversion(const bd_state_t* s, const bd_params_t* p, int64_t* result, void* stream) {
    return launch_op(s, p, OpArgs{OP_EDGE_INVERSION, 0, 0, 0.0, nullptr, nullptr, result}, s->tri.ne,
                     (cudaStream_t)stream);
}

int bd_tri_signed_area2(const bd_state_t* s, const bd_params_t* p, double* area, void* stream) {
    return launch_op(s, p, OpArgs{OP_SIGNED_AREA2, 0, 0, 0.0, nullptr, area, nullptr}, s->tri.nt,
                     (cudaStream_t)stream);
}

int bd_tri_delaunay_flags(const bd_state_t* s, const bd_params_t* p, uint8_t* flags, void* stream) {
    return launch_op(s, p, OpArgs{OP_DELAUNAY_FLAGS, 0, 0, 0.0, nullptr, flags, nullptr}, s->tri.ne,
                     (cudaStream_t)stream);
}

int bd_tri_inverted_edge_flags(const bd_state_t* s, const bd_params_t* p, uint8_t* flags, void* stream) {
    return launch_op(s, p, OpArgs{OP_INVERTED_FLAGS, 0, 0, 0.0, nullptr, flags, nullptr}, s->tri.ne,
                     (cudaStream_t)stream);
}

int bd_tri_flip_edges(const bd_state_t* s, const bd_params_t* p, const int64_t* edges, int64_t count,
                      int64_t* result, void* stream) {
    return launch_op(s, p, OpArgs{OP_FLIP_EDGES, count, 0, 0.0, edges, nullptr, result}, 1, (cudaStream_t)stream);
}

int bd_tri_repair_inversions(const bd_state_t* s, const bd_params_t* p, int64_t max_passes, int use_prev,
                             int64_t* result, void* stream) {
    return launch_op(s, p, OpArgs{OP_REPAIR, max_passes, use_prev, 0.0, nullptr, nullptr, result}, s->tri.ne,
                     (cudaStream_t)stream);
}

int bd_tri_restore_delaunay_ex(const bd_state_t* s, const bd_params_t* p, int64_t max_passes, int64_t* result,
                               void* stream) {
    return launch_op(s, p, OpArgs{OP_RESTORE, max_passes, 0, 0.0, nullptr, nullptr, result}, s->tri.ne,
                     (cudaStream_t)stream);
}

int bd_overlap_correct(const bd_state_t* s, const bd_params_t* p, int64_t n_pairs, int with_tri, int64_t* result,
                       void* stream) {
    return launch_op(s, p, OpArgs{OP_CORRECT_OVERLAPS, n_pairs, with_tri, 0.0, nullptr, nullptr, result}, n_pairs,
                     (cudaStream_t)stream);
}

int bd_tri_copy(const bd_tri_t* src, const bd_tri_t* dst, void* stream) {
    init_device_info();
    const int64_t items = src->ne > src->nt ? src->ne : src->nt;
    k_tri_copy<<<grid_for(items), 256, 0, (cudaStream_t)stream>>>(*src, *dst);
    return err_code(cudaGetLastError());
}

int bd_tri_audit_geometry(const bd_state_t* s, const bd_params_t* p, int64_t* out, void* stream) {
    init_device_info();
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(int64_t), st);
    if (e != cudaSuccess) return err_code(e);
    k_audit_geometry<<<grid_for(s->tri.ne), 256, 0, st>>>(s->tri, s->pos, p->L, p->tol, (unsigned long long*)out);
    return err_code(cudaGetLastError());
}

int64_t bd_tri_build_workspace_bytes(int64_t n, double L) { return n > 0 ? build_layout(n, L).total : 0; }

int bd_tri_build_initial(const double* pos, int64_t n, double L, const bd_tri_t* out, void* work, int64_t work_bytes,
                         int64_t* result, void* stream) {
    init_device_info();
    if (n < 3 || work_bytes < build_layout(n, L).total) return -(int)cudaErrorInvalidValue;
    cudaStream_t st = (cudaStream_t)stream;
    bd_tri_t o = *out;
    void* args[] = {(void*)&pos, (void*)&n, (void*)&L, (void*)&o, (void*)&work, (void*)&result};
    return coop_launch((const void*)k_tri_build_grid, n, args, st);
}

// FP64 FMA throughput probe (roofline denominator, bench.py): 8 independent
// DFMA chains per thread; *flops_out = flops issued by the launch
int bd_probe_fp64(int64_t iters, double* out, void* stream, double* flops_out) {
    init_device_info();
    const int nb = g_num_sms * 8;
    k_probe_fp64<<<nb, 256, 0, (cudaStream_t)stream>>>(iters, out);
    *flops_out = 2.0 * 8.0 * (double)iters * (double)nb * 256.0;
    return err_code(cudaGetLastError());
}

// ---- check of the branch-free IEEE sqrt / division of the EXACT kernel
// (bd_allpairs.cuh: sqrt_rn_inrange, div_rn_inrange) against sqrt() and '/'
// on n generated operand sets (tests/test_exact_fastpath_gpu.py).  Operands:
// random mantissas with exponents over the whole guarded range, perfect
// squares and products of short mantissas (exact roots and quotients) and
// one ulp either side of them, and the kernel's own shape num / (r2 sqrt(r2)).
// bad[0] = mismatches, bad[1..2] = the bits of the first offending operands,
// bad[3..6] = mismatches of sqrt, a / b, r2 sqrt(r2), num / den.
BD_DEV uint64_t probe_mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

BD_DEV double probe_make(uint64_t mant, int ex) {  // 1.mant * 2^ex
    return __longlong_as_double((long long)(((uint64_t)(ex + 1023) << 52) | (mant & 0xfffffffffffffull)));
}

BD_DEV void probe_cmp(double got, double want, double a, double b, unsigned long long* bad, int which) {
    if (dbits(got) != dbits(want)) {
        atomicAdd(&bad[3 + which], 1ull);
        if (atomicAdd(&bad[0], 1ull) == 0) {
            bad[1] = dbits(a);
            bad[2] = dbits(b);
        }
    }
}

__global__ void k_probe_exact_arith(uint64_t seed, int64_t n, unsigned long long* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t h1 = probe_mix(seed ^ (uint64_t)(3 * i)), h2 = probe_mix(seed ^ (uint64_t)(3 * i + 1));
        const uint64_t h3 = probe_mix(seed ^ (uint64_t)(3 * i + 2));
        const int ea = (int)(h3 % 401) - 200, eb = (int)((h3 >> 20) % 401) - 200;
        const int kind = (int)(h3 >> 40) & 7;
        const int ulps = (int)((h3 >> 44) & 3) - 1;  // -1, 0, +1, +2
        double a = probe_make(h1, ea), b = probe_make(h2, eb);
        if (kind == 1 || kind == 2) {  // short mantissas: exact squares / exact quotients (+- ulps)
            const double ra = probe_make(h1 & ~((1ull << 26) - 1), ea / 2);
            const double rb = probe_make(h2 & ~((1ull << 26) - 1), eb / 2);
            a = __longlong_as_double((long long)(dbits(ra * ra) + (int64_t)ulps));
            if (kind == 2) {
                b = rb;
                a = __longlong_as_double((long long)(dbits(ra * rb) + (int64_t)ulps));
            }
        } else if (kind == 3) {  // powers of two and all-ones mantissas
            a = probe_make((h1 & 1) ? 0ull : ~0ull, ea);
            b = probe_make((h2 & 1) ? 0ull : ~0ull, eb);
        }
        probe_cmp(sqrt_rn_inrange(a), sqrt(a), a, a, bad, 0);
        probe_cmp(div_rn_inrange(a, b), a / b, a, b, bad, 1);
        // the EXACT kernel's operands: num / (r2 sqrt(r2)), r2 from a square sum
        const double r2 = fabs(a) * 1e-100 < 1.0 ? fabs(a) : 1.0 / fabs(a);
        if (in_range(r2)) {
            const double den = r2 * sqrt_rn_inrange(r2);
            probe_cmp(den, r2 * sqrt(r2), r2, r2, bad, 2);
            probe_cmp(div_rn_inrange(b, den), b / den, b, den, bad, 3);
        }
    }
}

int bd_probe_exact_arith(uint64_t seed, int64_t n, void* bad, void* stream) {
    init_device_info();
    cudaMemsetAsync(bad, 0, 7 * sizeof(unsigned long long), (cudaStream_t)stream);
    k_probe_exact_arith<<<g_num_sms * 8, 256, 0, (cudaStream_t)stream>>>(seed, n, (unsigned long long*)bad);
    return err_code(cudaGetLastError());
}

// ---- grid-barrier probe (measurement only): latency of the cooperative
// grid.sync the step drivers end every phase with (tools/probe_barrier.py)
__global__ void k_probe_gridsync(int64_t iters, int mode, unsigned* bar) {
    for (int64_t i = 0; i < iters; ++i) cooperative_groups::this_grid().sync();
}

int bd_probe_barrier(int64_t iters, int mode, int ctas_per_sm, int threads, void* scratch, void* stream,
                     double* ms_out) {
    init_device_info();
    unsigned* bar = (unsigned*)scratch;  // [0, 256): barrier words + error count; from byte 256: a Ctl block
    cudaMemsetAsync(bar, 0, 256, (cudaStream_t)stream);
    void* args[] = {&iters, &mode, &bar};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, (cudaStream_t)stream);
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_probe_gridsync, dim3(g_num_sms * ctas_per_sm),
                                                dim3(threads), args, 0, (cudaStream_t)stream);
    cudaEventRecord(e1, (cudaStream_t)stream);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *ms_out = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return err_code(e);
}

int bd_timing_enable(int64_t launches) {
    for (cudaEvent_t e : g_tr.ev) cudaEventDestroy(e);
    g_tr.ev.assign(2 * (size_t)(launches > 0 ? launches : 0), nullptr);
    for (auto& e : g_tr.ev) cudaEventCreate(&e);
    g_tr.cap = launches > 0 ? launches : 0;
    g_tr.next = 0;
    return 0;
}

int64_t bd_timing_read(float* ms, int64_t max_n) {
    int64_t k = 0;
    for (; k < g_tr.next && k < max_n; ++k) {
        cudaEventSynchronize(g_tr.ev[2 * k + 1]);
        cudaEventElapsedTime(&ms[k], g_tr.ev[2 * k], g_tr.ev[2 * k + 1]);
    }
    return k;
}

const char* bd_build_info(void) {
    return "libbd_b200: sm_100a, -fmad=false (exact paths), TMA-staged all-pairs (exact + sorted fast), "
           "persistent cooperative step kernels (triangulation / Verlet)";
}

}  // extern "C"
