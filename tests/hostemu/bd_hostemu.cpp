// bd_hostemu.cpp -- TEST HARNESS: the product's step driver compiled for the host.
//
// Compiles paper_1703_02484_b200/csrc/bd_step.cuh (the exact source the GPU
// runs) with the ExecHost policy: one host thread walks every phase in
// order, barriers are no-ops.  This lets the CPU test suite check the
// driver's control flow and arithmetic (LFMIS flip selection, incidence
// gathers, rollback, crossings bookkeeping) against the oracle without a
// GPU.  It is loaded only by tests/; the product never uses it.
#include "../../paper_1703_02484_b200/csrc/bd_allpairs.cuh"
#include "../../paper_1703_02484_b200/csrc/bd_step.cuh"

using namespace bd;

extern "C" {

void bdh_prepare_params(bd_params_t* p) { prepare_params(p); }

int64_t bdh_workspace_bytes(int64_t n, int64_t ne, int64_t nt) { return ws_layout(n, ne, nt).total; }

double bdh_mi_fast(double d, const bd_params_t* p) { return mi_fast(d, p->L, p->mi_lo, p->mi_hi); }
double bdh_mi_ref(double d, double L) { return mi_ref(d, L); }

void bdh_normals(uint64_t seed, uint64_t stream, uint64_t call, uint64_t purpose, int64_t npairs, double* out) {
    for (int64_t i = 0; i < npairs; ++i) normal_pair(seed, stream, call, (uint64_t)i, purpose, out[2 * i], out[2 * i + 1]);
}

void bdh_long_range(const bd_state_t* s, const bd_params_t* p) {
    for (int64_t i = 0; i < p->n; ++i)
        lr_receiver_exact(s->pos, s->alpha, s->mu, p->n, p->L, p->mi_lo, p->mi_hi, i, s->force, s->force_err);
}

void bdh_step_tri(const bd_state_t* s, const bd_params_t* p, bd_stats_t* out) {
    bdh_long_range(s, p);
    Ctx c;
    c.p = *p;
    c.s = *s;
    c.w = ws_carve(s->work, p->n, s->tri.ne, s->tri.nt);
    c.call = *s->call;
    ExecHost x{c.w.ctl};
    step_tri_after_force(x, c, out);
}

int64_t bdh_restore_delaunay(const bd_state_t* s, const bd_params_t* p) {
    Ctx c;
    c.p = *p;
    c.s = *s;
    c.w = ws_carve(s->work, p->n, s->tri.ne, s->tri.nt);
    c.call = 0;
    ExecHost x{c.w.ctl};
    Red<ExecHost> R(x);
    for (int k = 0; k < 8; ++k) c.w.ctl->red[k] = 0;
    return restore_delaunay(x, R, c, 1000);
}

}  // extern "C"
