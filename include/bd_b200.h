/*
 * bd_b200.h -- C ABI of the B200-native Brownian-dynamics hot path.
 *
 * Drop-in boundary for the per-timestep path of the reference package
 * `brownsim` (arXiv 1703.02484 re-implementation, /root/reference/pkg).  The
 * reference has no formal plugin registry; its two de-facto boundaries are
 * (i) the kernel module brownsim._kernels (numpy arrays in, new arrays +
 * `err` sentinels out) and (ii) the simulation classes' step()/run().  Each
 * entry point below names the reference interface it replaces.
 *
 * Conventions
 *   - every pointer is a DEVICE pointer (cudaMalloc / torch CUDA storage)
 *     unless the name says _host; layouts are the reference's numpy layouts
 *     (positions (N,2) float64 row-major = interleaved x,y, int64 pair
 *     arrays, the six int32/int8 triangulation arrays);
 *   - calls are asynchronous on the given cudaStream_t (passed as void*);
 *     no entry point synchronises the host or allocates device memory;
 *     scratch comes from a caller-provided workspace sized by
 *     bd_workspace_bytes();
 *   - return value: 0 = launched OK, negative = CUDA launch error
 *     (-(cudaError_t)); simulation outcomes (singularity, non-convergence,
 *     rollback budget) are reported asynchronously in bd_stats_t.status.
 */
#ifndef BD_B200_H
#define BD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (bd_stats_t.status), mapped to the reference exceptions
 * core.py:18-45 by the Python layer */
#define BD_OK 0
#define BD_ERR_SINGULAR 1     /* SingularityError: zero separation (forces.py:55-58, :167-170) */
#define BD_ERR_NONCONV 2      /* NonConvergenceError (dynamics.py:131, :247; triangulation.py:329) */
#define BD_ERR_STEPFAIL 4     /* StepFailure: non-finite force / rollback budget (dynamics.py:84-86, :254-258) */
#define BD_ERR_FLIP 5         /* BrownsimError: unflippable edge (triangulation.py:261-280) */
#define BD_ERR_CAPACITY 6     /* a device buffer (Verlet pairs) is too small: host grows it and retries */
#define BD_ERR_BUILD 7        /* BuildError: no valid periodic triangulation (triangulation.py:545-550) */

/* force models of one step: long range (dynamics.py:194),
 * short range over a Verlet list, or their sum F_LR + F_SR */
#define BD_FORCE_LR 0
#define BD_FORCE_SR 1
#define BD_FORCE_LRSR 2

/* all-pairs arithmetic: EXACT reproduces _kernels.long_range_kernel bit for
 * bit; FAST uses fma + rsqrt/Newton (|dF|/|F| <= 1e-12) */
#define BD_LR_EXACT 0
#define BD_LR_FAST 1
/* FAST-SYM: FAST arithmetic with each unordered pair's r^-3 evaluated once
 * and applied to both directions (Newton's third law on the geometric
 * factor; csrc/bd_allpairs_sym.cuh).  Whole range only (shard it with
 * bd_force_sym_partial / _finish); workspace ~ n^2/64 bytes
 * (bd_long_range_workspace_bytes_for). */
#define BD_LR_FAST_SYM 2

/* PeriodicTriangulation arrays, triangulation.py:129-139 */
typedef struct bd_tri {
    int64_t nv, ne, nt;
    int32_t* tri_v;    /* (nt,3)   */
    int8_t* tri_shift; /* (nt,3,2) */
    int32_t* tri_edge; /* (nt,3)   */
    int32_t* edge_v;   /* (ne,2)   */
    int32_t* edge_tri; /* (ne,2)   */
    int8_t* edge_opp;  /* (ne,2)   */
} bd_tri_t;

/* SimParams (core.py:161-204) + run constants */
typedef struct bd_params {
    int64_t n;
    double L;
    double sigma, dt, diffusion, cap, clamp, r_cut, skin, tol;
    int64_t max_overlap_iters, max_rollbacks;
    uint64_t seed, stream;
    int64_t force_mode;   /* BD_FORCE_* */
    int64_t lr_precision; /* BD_LR_* */
    double mi_lo, mi_hi;  /* exact min-image breakpoints, filled by bd_prepare_params */
    double r_list;        /* Verlet list radius max(r_cut, sigma) + skin */
    int64_t ncx;          /* cells per axis of the Verlet grid (0 = all-pairs scan) */
    int64_t pair_capacity;/* capacity of the Verlet pair buffers */
    /* active Brownian particles (AbpState, dynamics.py:60-66, :349-399) */
    double abp_speed;         /* self-propulsion speed V0 */
    double abp_rot_diffusion; /* rotational diffusion D_r */
    int64_t abp_clamp_angle;  /* clamp the angular noise (clamp_angle_noise) */
} bd_params_t;

/* StepStats (dynamics.py:42-57) counters + error report */
typedef struct bd_stats {
    double dt_used;
    int64_t overlap_iterations, flip_passes, inversion_repairs, rollbacks, n_overlapping;
    int64_t status, err_i, err_k;
    int64_t rebuilds; /* Verlet rebuilds during this step */
    int64_t calls;    /* noise-call counter after this step (CounterRng.call; *s->call) */
    int64_t reserved[5];
    /* device work of the step, for the algorithmic-bytes roofline of the
     * O(N) path: passes of integrate, apply_crossings,
     * edge-inversion check, per-edge flag passes, per-triangle area passes,
     * independent-set rounds, flipped edges, overlap passes, overlap
     * gather/apply passes, incidence builds, Verlet rebuilds, short-range
     * force evaluations; then device time (ns) in maintenance, overlap
     * sweeps, incidence builds, the whole driver, Verlet rebuilds and
     * short-range forces; then spare words */
    int64_t work[24];
} bd_stats_t;

/* device state of one simulation */
typedef struct bd_state {
    double *pos, *prev, *force, *alpha, *mu; /* (n,2) (n,2) (n,2) (n,) (n,) */
    int64_t* force_err;                      /* (n,) err sentinels of the force kernels */
    int32_t* image;                          /* (n,2) unwrapped box images (MSD) */
    uint8_t* overlap_flags;                  /* (n,) last_overlap_flags */
    bd_tri_t tri;                            /* maintained triangulation */
    bd_tri_t tri_backup;                     /* rollback copy (triangulation.py:158-164) */
    uint64_t* call;                          /* noise call counter (1 element) */
    bd_stats_t* stats;                       /* device stats of the last step */
    /* Verlet list (forces.py:102-156): pairs, snapshot, count */
    int64_t* pair_a;
    int64_t* pair_b;
    double* vl_snap;
    int64_t* vl_meta; /* [0]=n_pairs, [1]=valid, [2]=rebuilds total, [3]=overlap candidates */
    void* work;       /* scratch of bd_workspace_bytes() bytes */
    int64_t work_bytes;
    double* angles;   /* (n,) ABP director angles (AbpState.angles), else NULL */
} bd_state_t;

/* fills p->mi_lo/mi_hi (and r_list/ncx) from p->L etc.; host-only helper */
void bd_prepare_params(bd_params_t* p);

/* scratch bytes of a simulation state: p (after bd_prepare_params: n, ncx,
 * pair_capacity) with ne edges / nt triangles (0, 0 without a triangulation) */
int64_t bd_workspace_bytes(const bd_params_t* p, int64_t ne, int64_t nt);

/* scratch bytes of the standalone pair-list entry points below
 * (bd_verlet_build, bd_short_range_forces, bd_overlap_pass) */
int64_t bd_pairs_workspace_bytes(int64_t n, double L, double r_list, int64_t n_pairs);

/* ---- kernel boundary (replaces brownsim._kernels) -------------------- */

/* long_range_kernel (_kernels.py:26-59): out[i] = sum_{k != i} mu_i alpha_k
 * r_ik / r^3 for receivers i in [i_begin, i_end) over all n sources;
 * err[i] = k+1 on a zero-separation pair (else 0). out/err index the full
 * range (rows outside [i_begin, i_end) are untouched). */
int bd_long_range_forces(const double* pos, const double* alpha, const double* mu, int64_t n,
                         double L, int64_t i_begin, int64_t i_end, int precision, double* out,
                         int64_t* err, void* work, void* stream);

/* scratch bytes of bd_long_range_forces (packed sources) for EXACT / FAST */
int64_t bd_long_range_workspace_bytes(int64_t n);

/* scratch bytes of bd_long_range_forces for a given precision (BD_LR_*) */
int64_t bd_long_range_workspace_bytes_for(int64_t n, int precision);

/* short_range_kernel (_kernels.py:62-91) over stored pairs, accumulated
 * per particle in ascending pair order (bit-exact). */
int bd_short_range_forces(const double* pos, const double* alpha, const double* mu, int64_t n,
                          const int64_t* pair_a, const int64_t* pair_b, int64_t n_pairs, double L,
                          double r_cut, double* out, int64_t* err, void* work, void* stream);

/* overlap_pass_kernel (_kernels.py:94-125): disp (n,2), flags (n,), count (1) */
int bd_overlap_pass(const double* pos, int64_t n, const int64_t* pair_a, const int64_t* pair_b,
                    int64_t n_pairs, double L, double sigma, double resolve, double* disp,
                    uint8_t* flags, int64_t* count, void* work, void* stream);

/* max_sq_displacement (_kernels.py:128-138) -> out[0] */
int bd_max_sq_displacement(const double* pos, const double* snap, int64_t n, double L, double* out,
                           void* stream);


/* build_cell_grid + cell_pairs (forces.py:81-99, _kernels.py:141-236):
 * ordered Verlet pair list identical to the reference's; writes count[0]
 * (pairs are written only when count <= capacity). */
int bd_verlet_build(const double* pos, int64_t n, double L, double r_list, int64_t* pair_a,
                    int64_t* pair_b, int64_t capacity, int64_t* count, void* work, void* stream);

/* brute_force_overlaps (_kernels.py:239-275), the O(N^2) debug oracle of
 * run(debug_scan=True): out[0] = number of pairs a < b closer than thresh,
 * out[1] = (a << 32) | b of the first such pair (or all ones) */
int bd_brute_overlaps(const double* pos, int64_t n, double L, double thresh, int64_t* out, void* stream);

/* counter-based normals for pairs [0, n_pairs) of one call */
int bd_normals(uint64_t seed, uint64_t stream_id, uint64_t call, uint64_t purpose, int64_t n_pairs,
               double* out, void* stream);

/* ---- simulation boundary (replaces LongRangeSimulation.step etc.) ---- */

/* the force evaluation of one step on the pre-move positions
 * (dynamics.py:194) for p->force_mode; writes s->force and s->force_err */
int bd_force(const bd_state_t* s, const bd_params_t* p, void* stream);

/* The same force in three calls, for sharding across GPUs (one process per
 * GPU, all holding the full state): every rank runs _prepare (sort + pack of
 * the sources), _slots for its own receiver slots [s0, s1) -- records
 * (fx, fy, flag) written to slot3[3*s .. 3*s+2] --, then the records of all
 * slots are all-gathered (NCCL) into one (n, 3) array and _finish scatters
 * them into s->force / s->force_err.  Slot order is the sorted order of the
 * FAST path and particle order for EXACT; each receiver's sum is computed
 * whole by one rank, so the result is bit-identical for every rank count. */
int bd_force_prepare(const bd_state_t* s, const bd_params_t* p, void* stream);
int bd_force_slots(const bd_state_t* s, const bd_params_t* p, int64_t s0, int64_t s1, double* slot3,
                   void* stream);
int bd_force_finish(const bd_state_t* s, const bd_params_t* p, const double* slot3, void* stream);

/* The FAST-SYM force (p->lr_precision == BD_LR_FAST_SYM) in two calls, for
 * sharding: every rank runs _sym_partial for its share of the circulant
 * block pairs (rank of world), writing the unscaled per-slot partial
 * P_r = A_r - B_r into part (n,2); the ranks all-reduce (sum) part (NCCL);
 * _sym_finish forms F = mu P and scatters it into s->force / s->force_err.
 * Deterministic for a given world size. */
int bd_force_sym_partial(const bd_state_t* s, const bd_params_t* p, int rank, int world, double* part,
                         void* stream);
int bd_force_sym_finish(const bd_state_t* s, const bd_params_t* p, const double* part, void* stream);

/* the FAST-SYM work split of rank `rank` of `world` (host only, no device
 * call): out[11] = {block slots B, blocks Mb, circulant half-range D,
 * chunks S, distances per chunk `per`, first chunk c0, chunk stride cs,
 * chunk count nch, 0, diagonal blocks [i0, i1)}.  Rank r owns the chunks
 * c = c0 + k cs (k < nch; dealt round-robin), i.e. every unordered block
 * pair (I, I + d mod Mb) with d in [1 + c per, 1 + (c + 1) per) (capped at
 * D; for even Mb, d = D only for I < Mb / 2), and the diagonal blocks I in
 * [i0, i1); together the ranks cover every unordered pair of slots exactly
 * once (the multi-GPU split of the prange over receivers, _kernels.py:37). */
int bd_sym_shard(int64_t n, int rank, int world, int64_t* out);

/* the rest of LongRangeSimulation.step after the force (dynamics.py:196-274):
 * integrate, pass-through check, inversion repair, Delaunay restoration,
 * overlap correction with the joint fixed point, rollback -- one persistent
 * kernel; StepStats counters to *out (device) */
int bd_maintain_tri(const bd_state_t* s, const bd_params_t* p, bd_stats_t* out, void* stream);

/* one LongRangeSimulation.step (dynamics.py:191-274) with the force model of
 * p->force_mode: force, integrate, pass-through check, inversion repair,
 * Delaunay restoration, overlap correction, rollback -- all on device. */
int bd_step_tri(const bd_state_t* s, const bd_params_t* p, void* stream);

/* `steps` consecutive steps, stats of step j written to stats_out[j]
 * (device array); stops at the first error. */
int bd_run_tri(const bd_state_t* s, const bd_params_t* p, int64_t steps, bd_stats_t* stats_out,
               void* stream);

/* one ShortRangeSimulation.step (dynamics.py:326-346): Verlet list kept
 * fresh on device, short-range force, integrate, overlap rounds over the
 * overlap candidates with rebuilds -- one persistent kernel */
int bd_step_verlet(const bd_state_t* s, const bd_params_t* p, bd_stats_t* stats_out, void* stream);

/* `steps` consecutive ShortRangeSimulation steps (stats_out[j], device) */
int bd_run_verlet(const bd_state_t* s, const bd_params_t* p, int64_t steps, bd_stats_t* stats_out,
                  void* stream);

/* one AbpSimulation.step (dynamics.py:368-399): Verlet list kept fresh,
 * ballistic move by V0 dt (cos theta, sin theta), angles += sqrt(2 D_r dt) xi
 * (xi = counter normals of one call, clamped if p->abp_clamp_angle), overlap
 * rounds over the candidates within sigma + skin -- one persistent kernel */
int bd_step_abp(const bd_state_t* s, const bd_params_t* p, bd_stats_t* stats_out, void* stream);

/* `steps` consecutive AbpSimulation steps (stats_out[j], device) */
int bd_run_abp(const bd_state_t* s, const bd_params_t* p, int64_t steps, bd_stats_t* stats_out, void* stream);

/* restore_delaunay (triangulation.py:319-334) on the state's triangulation
 * and positions; passes (or -1 on error) written to passes_out[0] (device) */
int bd_tri_restore_delaunay(const bd_state_t* s, const bd_params_t* p, int64_t* passes_out,
                            void* stream);

/* ---- method boundary: the pieces of a step, one call each ------------
 * The reference exposes the building blocks of a step as public functions
 * and PeriodicTriangulation methods, and its tests drive them one by one.
 * Each entry below runs the same device phase the fused step kernels use
 * (csrc/bd_ops.cuh) as one cooperative launch on the state `s` (positions
 * s->pos, previous positions s->prev, triangulation s->tri, scratch
 * s->work).  `result` is a small device int64 array, layout per call. */

/* dynamics.integrate (dynamics.py:73-94) with step dt: prev <- pos, then
 * pos = wrap((pos + F dt) + xi sqrt(D dt)), xi = counter normals of call
 * *s->call (which advances by one).  crossings (n,2) int64 (may be NULL);
 * result = {status (0 / BD_ERR_STEPFAIL: non-finite force, nothing moved),
 * particles that crossed, first bad particle} */
int bd_integrate(const bd_state_t* s, const bd_params_t* p, double dt, int64_t* crossings,
                 int64_t* result, void* stream);

/* dynamics.integrate (dynamics.py:73-94) with normals drawn by the caller:
 * noise (n,2) f64 standard normals -- e.g. the reference's own
 * rng.normals((n, 2)) (core.py:131-133, dynamics.py:89) -- clamped to
 * +-p->clamp on the device like clamped_normals (core.py:151-154); the call
 * counter *s->call is not touched.  Otherwise as bd_integrate. */
int bd_integrate_noise(const bd_state_t* s, const bd_params_t* p, double dt, const double* noise,
                       int64_t* crossings, int64_t* result, void* stream);

/* PeriodicTriangulation.apply_crossings (triangulation.py:166-177);
 * crossings (n,2) int64 */
int bd_tri_apply_crossings(const bd_state_t* s, const bd_params_t* p, const int64_t* crossings,
                           void* stream);

/* .edge_inversion_present(prev = s->prev, curr = s->pos) (triangulation.py:
 * 240-250); result[0] = 0 / 1 */
int bd_tri_edge_inversion(const bd_state_t* s, const bd_params_t* p, int64_t* result, void* stream);

/* .signed_area2(s->pos) (triangulation.py:186-191): area (nt,) float64 */
int bd_tri_signed_area2(const bd_state_t* s, const bd_params_t* p, double* area, void* stream);

/* .delaunay_flags(s->pos, tol = p->tol) (triangulation.py:226-229) and
 * .inverted_edge_flags(s->pos) (:231-234): flags (ne,) uint8 */
int bd_tri_delaunay_flags(const bd_state_t* s, const bd_params_t* p, uint8_t* flags, void* stream);
int bd_tri_inverted_edge_flags(const bd_state_t* s, const bd_params_t* p, uint8_t* flags, void* stream);

/* .flip_edge(e) (triangulation.py:254-302) for edges[0..count) in order;
 * result = {status (0 / BD_ERR_FLIP), index into edges of the failure} */
int bd_tri_flip_edges(const bd_state_t* s, const bd_params_t* p, const int64_t* edges, int64_t count,
                      int64_t* result, void* stream);

/* .repair_inversions(s->pos, prev = s->prev if use_prev else None,
 * max_passes) (triangulation.py:336-363);
 * result = {status, flips, passes, needs_rollback} (RepairResult) */
int bd_tri_repair_inversions(const bd_state_t* s, const bd_params_t* p, int64_t max_passes, int use_prev,
                             int64_t* result, void* stream);

/* .restore_delaunay(s->pos, tol = p->tol, max_passes) (triangulation.py:
 * 319-334); result = {status (0 / BD_ERR_NONCONV / BD_ERR_FLIP), passes} */
int bd_tri_restore_delaunay_ex(const bd_state_t* s, const bd_params_t* p, int64_t max_passes,
                               int64_t* result, void* stream);

/* dynamics.correct_overlaps (dynamics.py:97-133) over the fixed pair list
 * s->pair_a/pair_b[0..n_pairs); overlap participants OR-ed into
 * s->overlap_flags; with_tri: every sweep's crossings are applied to s->tri.
 * result = {status (0 / BD_ERR_NONCONV), sweeps}.  The workspace must be
 * sized with p->pair_capacity >= n_pairs. */
int bd_overlap_correct(const bd_state_t* s, const bd_params_t* p, int64_t n_pairs, int with_tri,
                       int64_t* result, void* stream);

/* save_state / restore_state (triangulation.py:158-164): copy the six
 * arrays of src into dst (same ne, nt) */
int bd_tri_copy(const bd_tri_t* src, const bd_tri_t* dst, void* stream);

/* clears the sticky error status of a state (after the host handled it) */
int bd_clear_status(const bd_state_t* s, void* stream);

/* geometric audit counters (triangulation.py:386-482): out[0] = triangles
 * with area2 <= 0, out[1] = edges violating the in-circle test */
int bd_tri_audit_geometry(const bd_state_t* s, const bd_params_t* p, int64_t* out, void* stream);

/* Initial periodic Delaunay triangulation (build_initial /
 * _build_from_tiling, triangulation.py:514-648) of the JITTERED points pos
 * (n,2) on the torus [0,L)^2, written into out (out->nt = 2n triangles,
 * out->ne = 3n edges, caller-allocated).  Same edge set as the reference's
 * build on the same jittered points; indexing by owner vertex (see
 * csrc/bd_build.cuh).  The caller then runs bd_tri_restore_delaunay on the
 * unjittered points and audits, as the reference does.  result (device
 * int64[4]) = {status (0 / BD_ERR_BUILD), vertex, reason, 0}; workspace of
 * bd_tri_build_workspace_bytes(n, L) bytes. */
int64_t bd_tri_build_workspace_bytes(int64_t n, double L);
int bd_tri_build_initial(const double* pos, int64_t n, double L, const bd_tri_t* out, void* work, int64_t work_bytes,
                         int64_t* result, void* stream);

/* library version / build info (host) */
/* measurement: record CUDA events around the next `launches` launches of
 * the all-pairs pair kernel (k_allpairs_sym), on the stream they are
 * launched on; bd_timing_read waits for them and writes each launch's device
 * time (ms) to ms[0..), returning how many.  bench.py's roofline of the
 * dominant kernel uses it.  Not thread-safe; off by default. */
int bd_timing_enable(int64_t launches);
int64_t bd_timing_read(float* ms, int64_t max_n);

const char* bd_build_info(void);

#ifdef __cplusplus
}
#endif

#endif /* BD_B200_H */
