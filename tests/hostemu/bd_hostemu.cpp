// bd_hostemu.cpp -- TEST HARNESS: the product's step drivers compiled for the host.
//
// Compiles paper_1703_02484_b200/csrc/bd_drivers.cuh (the exact source the
// GPU runs) with the ExecHost policy: one host thread walks every phase in
// order, barriers are no-ops.  This lets the CPU test suite check the
// drivers' control flow and arithmetic (LFMIS flip selection, incidence
// gathers, Verlet pair order, rollback, crossings bookkeeping) against the
// oracle without a GPU.  It is loaded only by tests/; the product never
// uses it.
#include "../../paper_1703_02484_b200/csrc/bd_allpairs.cuh"
#include "../../paper_1703_02484_b200/csrc/bd_drivers.cuh"
#include "../../paper_1703_02484_b200/csrc/bd_ops.cuh"
#include "../../paper_1703_02484_b200/csrc/bd_build.cuh"

using namespace bd;

static Ctx host_ctx(const bd_state_t* s, const bd_params_t* p) {
    Ctx c;
    c.p = *p;
    c.s = *s;
    c.w = ws_carve(s->work, *p, s->tri.ne, s->tri.nt);
    c.call = s->call ? *s->call : 0;
    ctx_init_work(c);
    return c;
}

extern "C" {

void bdh_prepare_params(bd_params_t* p) { prepare_params(p); }

int64_t bdh_workspace_bytes(const bd_params_t* p, int64_t ne, int64_t nt) { return ws_layout(*p, ne, nt).total; }

double bdh_mi_fast(double d, const bd_params_t* p) { return mi_fast(d, p->L, p->mi_lo, p->mi_hi); }
double bdh_mi_ref(double d, double L) { return mi_ref(d, L); }

void bdh_normals(uint64_t seed, uint64_t stream, uint64_t call, uint64_t purpose, int64_t npairs, double* out) {
    for (int64_t i = 0; i < npairs; ++i) normal_pair(seed, stream, call, (uint64_t)i, purpose, out[2 * i], out[2 * i + 1]);
}

void bdh_long_range(const bd_state_t* s, const bd_params_t* p) {
    for (int64_t i = 0; i < p->n; ++i)
        lr_receiver_exact(s->pos, s->alpha, s->mu, p->n, p->L, p->mi_lo, p->mi_hi, i, s->force, s->force_err);
}

// the selector form of the all-pairs loop (the GPU kernel's image decision)
void bdh_long_range_selector(const double* pos, const double* alpha, const double* mu, int64_t n,
                             const bd_params_t* p, double* out, int64_t* err) {
    for (int64_t i = 0; i < n; ++i)
        lr_receiver_selector(pos, alpha, mu, n, p->L, p->mi_lo, p->mi_hi, i, out, err);
}

void bdh_step_tri(const bd_state_t* s, const bd_params_t* p, bd_stats_t* out) {
    if (p->force_mode != BD_FORCE_SR) bdh_long_range(s, p);
    Ctx c = host_ctx(s, p);
    ExecHost x{c.w.ctl};
    step_tri_after_force(x, c, out);
}

void bdh_step_verlet(const bd_state_t* s, const bd_params_t* p, bd_stats_t* out) {
    Ctx c = host_ctx(s, p);
    ExecHost x{c.w.ctl};
    step_verlet(x, c, out);
}

void bdh_step_abp(const bd_state_t* s, const bd_params_t* p, bd_stats_t* out) {
    Ctx c = host_ctx(s, p);
    ExecHost x{c.w.ctl};
    step_abp(x, c, out);
}

int64_t bdh_restore_delaunay(const bd_state_t* s, const bd_params_t* p) {
    Ctx c = host_ctx(s, p);
    c.call = 0;
    ExecHost x{c.w.ctl};
    Red<ExecHost> R(x);
    for (int k = 0; k < 8; ++k) c.w.ctl->red[k] = 0;
    return restore_delaunay(x, R, c, 1000);
}

// Verlet build only (pairs into s->pair_a/pair_b); returns the pair count
int64_t bdh_verlet_build(const bd_state_t* s, const bd_params_t* p, double margin) {
    Ctx c = host_ctx(s, p);
    ExecHost x{c.w.ctl};
    Red<ExecHost> R(x);
    for (int k = 0; k < 8; ++k) c.w.ctl->red[k] = 0;
    c.w.ctl->status = 0;
    if (!vl_rebuild(x, R, c, margin)) return -1;
    return c.s.vl_meta[0];
}

// the method-boundary ops of csrc/bd_ops.cuh (op codes as in bd_capi.cu)
void bdh_op(const bd_state_t* s, const bd_params_t* p, int64_t op, int64_t i0, int64_t i1, double d0, const void* in,
            void* out, int64_t* res) {
    Ctx c = host_ctx(s, p);
    ExecHost x{c.w.ctl};
    switch (op) {
        case 1: op_integrate(x, c, d0, (int64_t*)out, res); break;
        case 2: op_apply_crossings(x, c, (const int64_t*)in); break;
        case 3: op_edge_inversion(x, c, res); break;
        case 4: op_signed_area2(x, c, (double*)out); break;
        case 5: op_edge_flags(x, c, false, (uint8_t*)out); break;
        case 6: op_edge_flags(x, c, true, (uint8_t*)out); break;
        case 7: op_flip_edges(x, c, (const int64_t*)in, i0, res); break;
        case 8: op_repair_inversions(x, c, i0, i1 != 0, res); break;
        case 9: op_restore_delaunay(x, c, i0, res); break;
        case 10: op_correct_overlaps(x, c, i0, i1 != 0, res); break;
        default: break;
    }
}

// image selector of one coordinate (bd_allpairs.cuh axis_select): out = {T, shift_le, shift_gt, amb}
void bdh_axis_select(double xi, double L, double lo, double hi, uint64_t* T, double* shifts, int* amb) {
    const AxisSel a = axis_select(xi, L, lo, hi);
    *T = a.T;
    shifts[0] = a.shift_le;
    shifts[1] = a.shift_gt;
    *amb = a.amb;
}

int64_t bdh_tri_build_workspace_bytes(int64_t n, double L) { return build_layout(n, L).total; }

void bdh_tri_build(const double* pos, int64_t n, double L, const bd_tri_t* out, void* work, int64_t* res) {
    BuildCtx c;
    c.g = build_geo(n, L);
    c.w = build_carve(work, n, L);
    c.pos = pos;
    c.out = *out;
    ExecHost x{c.w.ctl};
    static Poly P, Q;
    tri_build(x, c, P, Q, res);
}

}  // extern "C"
