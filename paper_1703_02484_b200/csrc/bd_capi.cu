// bd_capi.cu -- extern "C" entry points of libbd_b200.so (include/bd_b200.h).
//
// Host side only launches: every loop of the step runs inside the
// persistent step kernel (bd_step.cuh) or the all-pairs kernel
// (bd_allpairs.cuh).  No entry point allocates device memory or
// synchronises the host.
#include <cuda_runtime.h>

#include <mutex>

#include "bd_allpairs.cuh"
#include "bd_step.cuh"

using namespace bd;

namespace {

constexpr int LR_BT = 128;  // receivers per CTA of the all-pairs kernel
constexpr int LR_TS = 512;  // sources per smem stage (2 stages x 16 KiB)
constexpr int STEP_BT = 256;
constexpr int BLOCK_BT = 1024;

int g_num_sms = 0;
int g_grid_blocks_per_sm = 0;
std::once_flag g_once;

int64_t block_max_n() {
    static int64_t v = -1;
    if (v < 0) {
        const char* e = getenv("BD_BLOCK_MAX_N");
        v = e ? atoll(e) : 4096;
    }
    return v;
}

__global__ void __launch_bounds__(STEP_BT) k_step_tri_grid(bd_state_t s, bd_params_t p, bd_stats_t* out) {
    Ctx c;
    c.p = p;
    c.s = s;
    c.w = ws_carve(s.work, p.n, s.tri.ne, s.tri.nt);
    c.call = *s.call;
    ExecGrid x{c.w.ctl};
    step_tri_after_force(x, c, out);
}

__global__ void __launch_bounds__(BLOCK_BT) k_step_tri_block(bd_state_t s, bd_params_t p, bd_stats_t* out) {
    Ctx c;
    c.p = p;
    c.s = s;
    c.w = ws_carve(s.work, p.n, s.tri.ne, s.tri.nt);
    c.call = *s.call;
    ExecBlock x{c.w.ctl};
    step_tri_after_force(x, c, out);
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
    Ctx c;
    c.p = p;
    c.s = s;
    c.w = ws_carve(s.work, p.n, s.tri.ne, s.tri.nt);
    c.call = 0;
    ExecGrid x{c.w.ctl};
    restore_delaunay_entry(x, c, out);
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

void init_device_info() {
    std::call_once(g_once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        int nb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_step_tri_grid, STEP_BT, 0);
        int nb2 = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb2, k_restore_delaunay_grid, STEP_BT, 0);
        g_grid_blocks_per_sm = nb < nb2 ? nb : nb2;
        if (g_grid_blocks_per_sm < 1) g_grid_blocks_per_sm = 1;
        cudaFuncSetAttribute(k_lr_tiled<false, LR_BT, LR_TS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             2 * LR_TS * 32);
        cudaFuncSetAttribute(k_lr_tiled<true, LR_BT, LR_TS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             2 * LR_TS * 32);
    });
}

int grid_blocks(int64_t work_items) {
    int64_t want = (work_items + STEP_BT - 1) / STEP_BT;
    int64_t cap = (int64_t)g_num_sms * g_grid_blocks_per_sm;
    if (cap > 4096) cap = 4096;
    if (want > cap) want = cap;
    return (int)(want < 1 ? 1 : want);
}

int err_code(cudaError_t e) { return e == cudaSuccess ? 0 : -(int)e; }

int launch_lr(const double4* src, const double* mu, int64_t n, const bd_params_t& p, int64_t i0, int64_t i1,
              int precision, double* out, int64_t* err, cudaStream_t st) {
    if (i1 <= i0) return 0;
    const int64_t nb = (i1 - i0 + LR_BT - 1) / LR_BT;
    const size_t smem = 2 * LR_TS * 32;
    if (precision == BD_LR_FAST) {
        k_lr_tiled<true, LR_BT, LR_TS><<<(unsigned)nb, LR_BT, smem, st>>>(src, mu, n, p.L, p.mi_lo, p.mi_hi, i0, i1,
                                                                          out, err);
        k_lr_rescan<<<(unsigned)((i1 - i0 + 255) / 256 < 1184 ? (i1 - i0 + 255) / 256 : 1184), 256, 0, st>>>(
            src, n, p.L, p.mi_lo, p.mi_hi, i0, i1, err);
    } else {
        k_lr_tiled<false, LR_BT, LR_TS><<<(unsigned)nb, LR_BT, smem, st>>>(src, mu, n, p.L, p.mi_lo, p.mi_hi, i0,
                                                                           i1, out, err);
    }
    return err_code(cudaGetLastError());
}

int launch_pack(const double* pos, const double* alpha, int64_t n, double4* src, cudaStream_t st) {
    int64_t nb = (n + 255) / 256;
    if (nb > 4096) nb = 4096;
    if (nb < 1) nb = 1;
    k_pack_sources<<<(unsigned)nb, 256, 0, st>>>(pos, alpha, n, src);
    return err_code(cudaGetLastError());
}

int launch_force(const bd_state_t* s, const bd_params_t* p, cudaStream_t st) {
    init_device_info();
    const Ws w = ws_carve(s->work, p->n, s->tri.ne, s->tri.nt);
    // force on the pre-move positions (dynamics.py:194)
    int rc = launch_pack(s->pos, s->alpha, p->n, (double4*)w.src4, st);
    if (rc) return rc;
    return launch_lr((const double4*)w.src4, s->mu, p->n, *p, 0, p->n, (int)p->lr_precision, s->force,
                     s->force_err, st);
}

int launch_maintain_tri(const bd_state_t* s, const bd_params_t* p, bd_stats_t* out, cudaStream_t st) {
    init_device_info();
    bd_state_t sv = *s;
    bd_params_t pv = *p;
    if (p->n <= block_max_n()) {
        k_step_tri_block<<<1, BLOCK_BT, 0, st>>>(sv, pv, out);
        return err_code(cudaGetLastError());
    }
    const int64_t items = s->tri.ne > p->n ? s->tri.ne : p->n;
    void* args[] = {&sv, &pv, &out};
    return err_code(cudaLaunchCooperativeKernel((const void*)k_step_tri_grid, dim3(grid_blocks(items)), dim3(STEP_BT),
                                                args, 0, st));
}

int launch_step_tri(const bd_state_t* s, const bd_params_t* p, bd_stats_t* out, cudaStream_t st) {
    int rc = launch_force(s, p, st);
    if (rc) return rc;
    return launch_maintain_tri(s, p, out, st);
}

}  // namespace

extern "C" {

void bd_prepare_params(bd_params_t* p) { prepare_params(p); }

int64_t bd_workspace_bytes(int64_t n, int64_t ne, int64_t nt, int64_t pair_capacity) {
    (void)pair_capacity;
    return ws_layout(n, ne, nt).total;
}

int64_t bd_long_range_workspace_bytes(int64_t n) { return 32 * n + 256; }

int bd_long_range_forces(const double* pos, const double* alpha, const double* mu, int64_t n, double L, int64_t i_begin,
                         int64_t i_end, int precision, double* out, int64_t* err, void* work, void* stream) {
    init_device_info();
    cudaStream_t st = (cudaStream_t)stream;
    bd_params_t p;
    memset(&p, 0, sizeof(p));
    p.L = L;
    bd_prepare_params(&p);
    int rc = launch_pack(pos, alpha, n, (double4*)work, st);
    if (rc) return rc;
    return launch_lr((const double4*)work, mu, n, p, i_begin, i_end, precision, out, err, st);
}

int bd_normals(uint64_t seed, uint64_t stream_id, uint64_t call, uint64_t purpose, int64_t n_pairs, double* out,
               void* stream) {
    int64_t nb = (n_pairs + 255) / 256;
    if (nb > 4096) nb = 4096;
    if (nb < 1) nb = 1;
    k_normals<<<(unsigned)nb, 256, 0, (cudaStream_t)stream>>>(seed, stream_id, call, purpose, n_pairs, out);
    return err_code(cudaGetLastError());
}

int bd_force(const bd_state_t* s, const bd_params_t* p, void* stream) {
    return launch_force(s, p, (cudaStream_t)stream);
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

int bd_clear_status(const bd_state_t* s, void* stream) {
    const Ws w = ws_carve(s->work, 0, 0, 0);
    return err_code(cudaMemsetAsync(&w.ctl->status, 0, 3 * sizeof(unsigned long long), (cudaStream_t)stream));
}

int bd_tri_restore_delaunay(const bd_state_t* s, const bd_params_t* p, int64_t* passes_out, void* stream) {
    init_device_info();
    bd_state_t sv = *s;
    bd_params_t pv = *p;
    void* args[] = {&sv, &pv, &passes_out};
    const int64_t items = s->tri.ne > p->n ? s->tri.ne : p->n;
    return err_code(cudaLaunchCooperativeKernel((const void*)k_restore_delaunay_grid, dim3(grid_blocks(items)),
                                                dim3(STEP_BT), args, 0, (cudaStream_t)stream));
}

int bd_tri_audit_geometry(const bd_state_t* s, const bd_params_t* p, int64_t* out, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(out, 0, 2 * sizeof(int64_t), st);
    if (e != cudaSuccess) return err_code(e);
    int64_t items = s->tri.ne;
    int64_t nb = (items + 255) / 256;
    if (nb > 4096) nb = 4096;
    if (nb < 1) nb = 1;
    k_audit_geometry<<<(unsigned)nb, 256, 0, st>>>(s->tri, s->pos, p->L, p->tol, (unsigned long long*)out);
    return err_code(cudaGetLastError());
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

const char* bd_build_info(void) {
    return "libbd_b200: sm_100a, -fmad=false (exact paths), TMA bulk all-pairs, cooperative step kernel";
}

}  // extern "C"
