"""Step loops on the GPU, with the reference's API.

LongRangeSimulation and ShortRangeSimulation mirror brownsim.dynamics
(dynamics.py:177-346): constructors (sys, params, rng, ...), step() ->
StepStats, run(steps, on_step) -> list[StepStats], state read-out via .sys,
.tri, .last_overlap_flags, .step_index, .rebuilds.

A long-range step is two launches on the current CUDA stream: the all-pairs
force kernel and ONE persistent cooperative kernel that runs integrate, the
pass-through check, inversion repair, Delaunay flips, overlap correction,
the joint fixed point and the rollback loop entirely on the device
(csrc/bd_drivers.cuh).  A short-range step is one persistent kernel (Verlet
list maintenance, short-range force, integrate, overlap rounds).  The host
reads back only the StepStats counters (16 words per step, once per run()).

Extra keyword arguments of LongRangeSimulation (not in the reference):
  force        "long-range" (default), "short-range" or "long+short" -- the
               composite force models of SURVEY.md §0 (Verlet-list short range
               with params.r_cutoff); the triangulation stays the overlap
               neighbour provider in every case;
  precision    "exact" (bit-identical to the reference), "fast-sym" (FAST
               arithmetic, each unordered pair's r^-3 evaluated once for both
               directions; sharded by block pairs + all-reduce; workspace
               ~ n^2/64 bytes: 18 GB at 1M particles), "auto" (exact up to
               4,096 particles, then fast-sym while that fits half the free
               HBM, else fast) or "fast" (sorted,
               FMA + rsqrt all-pairs; |dF|/|F| ~1e-13);
  skin         Verlet skin for the short-range force (default sigma / 2).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._hostview import HostView, Versioned
from ._lib import check, lib, require_cuda
from .core import (BrownsimError, CounterRng, NonConvergenceError, ParticleSystem, SimParams, SingularityError,
                   StepFailure)
from .forces import verlet_pair_capacity
from .triangulation import TRI_KEYS, PeriodicTriangulation

RESOLVE_FRAC = 1.0 - 1e-9  # dynamics.py:39

FORCE_MODES = {"long-range": _abi.BD_FORCE_LR, "short-range": _abi.BD_FORCE_SR, "long+short": _abi.BD_FORCE_LRSR}
PRECISIONS = {"exact": _abi.BD_LR_EXACT, "fast": _abi.BD_LR_FAST, "fast-sym": _abi.BD_LR_FAST_SYM}
AUTO_SYM_FREE_FRACTION = 0.5  # precision="auto": FAST-SYM while its workspace (~n^2/64 B) fits half the free HBM
AUTO_EXACT_MAX_N = 4096  # precision="auto": EXACT up to here (B200: 0.033 ms at 1,024 vs 0.17 for FAST-SYM's launch chain)


@dataclass
class StepStats:
    """Per-step counters and phase timings (dynamics.py:42-57)."""

    step: int
    dt_used: float
    overlap_iterations: int = 0
    flip_passes: int = 0
    inversion_repairs: int = 0
    rollbacks: int = 0
    n_overlapping: int = 0
    force_ms: float = 0.0
    maintain_ms: float = 0.0
    overlap_ms: float = 0.0
    step_ms: float = 0.0
    overlap_flags: np.ndarray | None = field(default=None, repr=False)
    # device work counters of the step (not in the reference; csrc/bd_step.cuh WK_*, roofline.py)
    work: dict | None = field(default=None, repr=False)


from .validation import MissedOverlapError  # noqa: E402  (dynamics.py:69-70)


def _tri_struct(tensors: dict, nv: int) -> _abi.BdTri:
    return _abi.BdTri(nv, int(tensors["edge_v"].shape[0]), int(tensors["tri_v"].shape[0]),
                      *[tensors[k].data_ptr() for k in TRI_KEYS])


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def make_params(params: SimParams, box_length: float, seed: int, stream: int, force_mode: int = 0,
                precision: int = 0, skin: float | None = None, pairs: bool = False,
                no_cutoff: bool = False) -> _abi.BdParams:
    p = _abi.BdParams()
    p.n = params.n
    p.L = float(box_length)
    p.sigma, p.dt, p.diffusion = float(params.sigma), float(params.dt), float(params.diffusion)
    p.cap, p.clamp = float(params.displacement_cap), float(params.noise_clamp)
    p.r_cut = float(params.r_cutoff) if params.r_cutoff is not None and not no_cutoff else 0.0
    p.skin = 0.5 * params.sigma if skin is None else float(skin)
    p.tol = 1e-12
    p.max_overlap_iters, p.max_rollbacks = int(params.max_overlap_iters), int(params.max_rollbacks)
    p.seed, p.stream = int(seed) & ((1 << 64) - 1), int(stream) & ((1 << 64) - 1)
    p.force_mode, p.lr_precision = int(force_mode), int(precision)
    lib().bd_prepare_params(ctypes.byref(p))  # mi breakpoints, r_list, ncx
    p.pair_capacity = verlet_pair_capacity(params.n, box_length, p.r_list, params.sigma) if pairs else 0
    return p


class _Engine:
    """Device buffers + the C-ABI state struct of one simulation."""

    def __init__(self, sys: ParticleSystem, tri: PeriodicTriangulation | None, bparams: _abi.BdParams, call: int):
        torch = require_cuda()
        dev = sys.device
        n = sys.n
        self.sys, self.tri, self.p = sys, tri, bparams
        self.force_err = torch.zeros(n, dtype=torch.int64, device=dev)
        self.overlap_flags = torch.zeros(n, dtype=torch.uint8, device=dev)
        self.call_t = torch.tensor([call], dtype=torch.int64, device=dev)
        self.stats_t = torch.zeros(_abi.STATS_WORDS, dtype=torch.int64, device=dev)
        cap = int(bparams.pair_capacity)
        self.pair_a = torch.zeros(max(cap, 1), dtype=torch.int64, device=dev)
        self.pair_b = torch.zeros(max(cap, 1), dtype=torch.int64, device=dev)
        self.vl_snap = torch.zeros((n, 2), dtype=torch.float64, device=dev)
        self.vl_meta = torch.zeros(8, dtype=torch.int64, device=dev)
        ne = tri.n_edges if tri is not None else 0
        nt = tri.n_triangles if tri is not None else 0
        wb = lib().bd_workspace_bytes(ctypes.byref(bparams), ne, nt)
        self.work = torch.zeros(wb // 8 + 64, dtype=torch.int64, device=dev)
        s = _abi.BdState()
        s.pos, s.prev, s.force = sys.positions_t.data_ptr(), sys.positions_prev_t.data_ptr(), sys.forces_t.data_ptr()
        s.alpha, s.mu = sys.alpha_t.data_ptr(), sys.mu_t.data_ptr()
        s.force_err = self.force_err.data_ptr()
        s.image = sys.image_t.data_ptr()
        s.overlap_flags = self.overlap_flags.data_ptr()
        if tri is not None:
            s.tri = _tri_struct(tri.tensors(), n)
            s.tri_backup = _tri_struct(tri.backup_tensors(), n)
        s.call = self.call_t.data_ptr()
        s.stats = self.stats_t.data_ptr()
        s.pair_a, s.pair_b = self.pair_a.data_ptr(), self.pair_b.data_ptr()
        s.vl_snap, s.vl_meta = self.vl_snap.data_ptr(), self.vl_meta.data_ptr()
        s.work = self.work.data_ptr()
        s.work_bytes = self.work.numel() * 8
        self.s = s

    def clear_status(self):
        check(lib().bd_clear_status(ctypes.byref(self.s), _stream()), "bd_clear_status")


def _check_rng(rng):
    """The device draws counter-based noise, so `rng` must be
    a CounterRng.  The reference's RngStream (numpy Philox + ziggurat,
    core.py:111-139) is not counter-addressable: name the replacement."""
    if all(hasattr(rng, k) for k in ("seed", "stream", "call")):
        return
    if hasattr(rng, "seed") and hasattr(rng, "stream"):
        raise BrownsimError(
            f"rng {type(rng).__name__}(seed={rng.seed}, stream={rng.stream}) draws numpy ziggurat normals, which the "
            f"device cannot reproduce; pass paper_1703_02484_b200.CounterRng({rng.seed}, {rng.stream}) instead "
            f"(same key; the reference replays its normals with oracle.noise_np.CounterNormals({rng.seed}, "
            f"{rng.stream}))")
    raise BrownsimError("the device noise is counter-based: rng must be a CounterRng(seed, stream[, call])")


def _rng_counter(rng):
    _check_rng(rng)
    return int(rng.seed) & ((1 << 64) - 1), int(rng.stream) & ((1 << 64) - 1), int(rng.call)


def integrate(sys: ParticleSystem, forces, params: SimParams, rng, dt: float | None = None) -> np.ndarray:
    """dynamics.py:73-94 on the GPU: one Euler-Maruyama update of all
    positions (prev <- pos; pos = wrap((pos + F dt) + xi sqrt(D dt)), xi the
    +-noise_clamp clamped normals); returns the box crossings (N, 2) int64.
    Non-finite forces raise StepFailure before anything moves.

    With a CounterRng, xi are the counter normals of call rng.call (drawn
    on the device; the call advances by one).  Any other rng with the
    reference's `normals(shape, dtype)` method -- e.g. the reference's own
    numpy RngStream -- is asked for one (N, 2) block exactly like the
    reference does (dynamics.py:89), which is uploaded and used instead."""
    import torch
    from ._ops import OpState, as_device
    if dt is None:
        dt = params.dt
    n = sys.n
    f = as_device(forces, torch.float64, sys.device, (n, 2))
    op = OpState(n, sys.box.length, sys.device)
    op.p.diffusion, op.p.clamp, op.p.sigma = float(params.diffusion), float(params.noise_clamp), float(params.sigma)
    cross = torch.zeros((n, 2), dtype=torch.int64, device=sys.device)
    op.bind(pos=sys.positions_t, prev=sys.positions_prev_t, force=f, image=sys.image_t)
    counter = all(hasattr(rng, k) for k in ("seed", "stream", "call"))
    if counter:
        seed, stream, call = _rng_counter(rng)
        op.p.seed, op.p.stream = seed, stream
        op.call_t.fill_(call)
    else:
        if not torch.isfinite(f).all():  # the reference checks before it draws (dynamics.py:84-86)
            bad = int((~torch.isfinite(f).all(dim=1)).nonzero()[0, 0].item())
            raise StepFailure(f"non-finite force on particle {bad}")
        xi = as_device(np.ascontiguousarray(rng.normals((n, 2), dtype=np.float64), dtype=np.float64),
                       torch.float64, sys.device, (n, 2))
    sys.bump_version()
    if counter:
        res = op.run("bd_integrate", ctypes.c_double(float(dt)), ctypes.c_void_p(cross.data_ptr()), op.res_ptr)
    else:
        res = op.run("bd_integrate_noise", ctypes.c_double(float(dt)), ctypes.c_void_p(xi.data_ptr()),
                     ctypes.c_void_p(cross.data_ptr()), op.res_ptr)
    if res[0] == _abi.BD_ERR_STEPFAIL:
        raise StepFailure(f"non-finite force on particle {int(res[2])}")
    if counter:
        rng.call = call + 1
    return cross.cpu().numpy()


def correct_overlaps(sys: ParticleSystem, pair_a, pair_b, params: SimParams, tri: PeriodicTriangulation | None = None,
                     flags_out: np.ndarray | None = None) -> int:
    """dynamics.py:97-133 on the GPU: push overlapping pairs of the fixed
    list apart (per-particle sums in ascending pair order, displacement
    capped at params.displacement_cap, wrap) until none remain; with `tri`
    every sweep's crossings are applied to it.  Returns the sweeps that
    corrected something; NonConvergenceError after max_overlap_iters."""
    import torch
    from ._ops import OpState, as_device
    pa = as_device(pair_a, torch.int64, sys.device).reshape(-1)
    pb = as_device(pair_b, torch.int64, sys.device).reshape(-1)
    m = int(pa.numel())
    n = sys.n
    op = OpState(n, sys.box.length, sys.device, tri=tri, n_pairs=max(m, 1), sigma=params.sigma)
    op.p.cap = float(params.displacement_cap)
    op.p.max_overlap_iters = int(params.max_overlap_iters)
    flags = torch.zeros(n, dtype=torch.uint8, device=sys.device)
    op.bind(pos=sys.positions_t, pair_a=pa, pair_b=pb, overlap_flags=flags, image=sys.image_t)
    sys.bump_version()
    if tri is not None:
        tri.bump_version()
    res = op.run("bd_overlap_correct", m, int(tri is not None), op.res_ptr)
    if flags_out is not None:
        flags_out |= flags.cpu().numpy().astype(bool)
    if res[0] == _abi.BD_ERR_NONCONV:
        raise NonConvergenceError(f"overlap correction still unresolved after {params.max_overlap_iters} sweeps")
    if res[0]:
        raise BrownsimError(f"correct_overlaps: device status {int(res[0])}")
    return int(res[1])


def _raise_for(st: dict, step_index: int):
    code = int(st["status"])
    if code == _abi.BD_OK:
        return
    if code == _abi.BD_ERR_SINGULAR:
        raise SingularityError(f"particles {st['err_i']} and {st['err_k']} at zero separation")
    if code == _abi.BD_ERR_NONCONV:
        raise NonConvergenceError(f"step {step_index}: iterative procedure exceeded its iteration cap")
    if code == _abi.BD_ERR_STEPFAIL:
        raise StepFailure(f"step {step_index}: non-finite force or rollback budget exhausted "
                          f"(particle/rollbacks {st['err_i']})")
    if code == _abi.BD_ERR_FLIP:
        raise BrownsimError(f"step {step_index}: edge {st['err_i']} not flippable")
    if code == _abi.BD_ERR_CAPACITY:
        raise BrownsimError(f"step {step_index}: Verlet list of {st['err_i']} pairs exceeds capacity {st['err_k']}")
    raise BrownsimError(f"step {step_index}: device status {code}")


def _decode_stats(words: np.ndarray) -> dict:
    raw = _abi.BdStats.from_buffer_copy(np.ascontiguousarray(words, dtype=np.int64).tobytes())
    d = {k: getattr(raw, k) for k, _ in _abi.BdStats._fields_ if k not in ("reserved", "work")}
    d["work"] = {k: int(raw.work[i]) for i, k in enumerate(_abi.WORK_KEYS)}
    return d


def _phase_ms(work: dict, force_ev_ms: float, drv_ms: float, tri: bool) -> tuple:
    """StepStats (force_ms, maintain_ms, overlap_ms) with the reference's
    meanings (dynamics.py:193-270, :328-341), from the device phase timers of
    the step kernel (bd_stats_t.work, %globaltimer) and the force launch's
    event time.  Triangulation steps: maintain = pass-through check +
    inversion repair + Delaunay restoration, overlap = overlap rounds (with
    their pair-incidence builds).  Verlet steps: maintain = list rebuild,
    force = short-range force, overlap = integrate + overlap rounds."""
    ns = lambda k: float(work.get(k, 0)) * 1e-6
    if tri:
        return force_ev_ms + ns("t_sr_force_ns"), ns("t_maintain_ns"), ns("t_overlap_ns") + ns("t_incidence_ns")
    verlet, sr = ns("t_verlet_ns"), ns("t_sr_force_ns")
    return sr, verlet, max(drv_ms - verlet - sr, 0.0)


class _SimulationBase:
    """Shared run loop (dynamics.py:149-174); subclasses provide the launches."""

    _two_phase = False  # force kernel + driver kernel (timed separately)

    def __init__(self, sys: ParticleSystem, params: SimParams, rng, debug_scan=False, collect_flags=False):
        self.sys = sys
        self.params = params
        self.rng = rng if rng is not None else CounterRng(0, 2)
        _check_rng(self.rng)
        self.debug_scan = debug_scan
        self.collect_flags = collect_flags
        self.step_index = 0

    @property
    def last_overlap_flags(self) -> np.ndarray:
        return self._eng.overlap_flags.cpu().numpy().astype(bool)

    @property
    def rebuilds(self) -> int:
        return int(self._eng.vl_meta[2].item())

    def _refresh_params(self):
        # the reference lets callers mutate sim.params between steps (e.g. dt)
        p, b = self.params, self.bparams
        b.dt, b.diffusion = float(p.dt), float(p.diffusion)
        b.max_overlap_iters, b.max_rollbacks = int(p.max_overlap_iters), int(p.max_rollbacks)
        b.cap, b.clamp = float(p.displacement_cap), float(p.noise_clamp)

    def step(self) -> StepStats:
        return self.run(1)[0]

    def run(self, steps: int, on_step=None) -> list:
        """`steps` steps; without on_step / debug_scan / collect_flags they are
        queued back to back with a single host synchronisation at the end."""
        self._refresh_params()
        if steps <= 0:
            return []
        self._eng.clear_status()
        if on_step is None and not self.debug_scan and not self.collect_flags:
            return self._run_batch(steps)
        out = []
        for _ in range(steps):
            out.extend(self._run_batch(1))
            if self.debug_scan:
                from .validation import debug_overlap_scan
                debug_overlap_scan(self.sys, self.params)
            if on_step is not None:
                on_step(self, out[-1])
        return out

    def _bump_versions(self):
        self.sys.bump_version()
        if getattr(self, "tri", None) is not None:
            self.tri.bump_version()
        if getattr(self, "abp", None) is not None:
            self.abp.bump_version()

    def _launch_force(self):
        pass

    def _launch_driver(self, stats_ptr: int):
        raise NotImplementedError

    def _run_batch(self, steps: int) -> list:
        import torch
        self._bump_versions()  # host copies read before these steps go stale
        # per-call buffers are kept (a step() per host round trip stays lean):
        # the stats rows (every launch writes its row's status word first thing)
        # and the timing events
        cache = self.__dict__.setdefault("_batch_cache", {})
        stats = cache.get(("stats", steps))
        if stats is None:
            stats = cache[("stats", steps)] = torch.zeros((steps, _abi.STATS_WORDS), dtype=torch.int64,
                                                          device=self.sys.device)
            cache[("host", steps)] = torch.empty((steps, _abi.STATS_WORDS), dtype=torch.int64).pin_memory()
        host_t = cache[("host", steps)]
        evs = cache.setdefault("events", [])
        while len(evs) < 2 * steps + 2:
            evs.append(torch.cuda.Event(enable_timing=True))
        evs[0].record()
        for j in range(steps):
            self._launch_force()
            evs[2 * j + 1].record()
            self._launch_driver(stats[j].data_ptr())
            evs[2 * j + 2].record()
        host_t.copy_(stats, non_blocking=True)
        evs[2 * steps + 1].record()
        evs[2 * steps + 1].synchronize()
        host = host_t.numpy()
        decoded = [_decode_stats(host[j]) for j in range(steps)]
        # the noise-call counter after the batch: from the last step's stats
        # when every step ran clean (no second device read), else from HBM
        if all(d["status"] == 0 for d in decoded):
            self.rng.call = int(decoded[-1]["calls"])
        else:
            self.rng.call = int(self._eng.call_t.item())
        res = []
        for j in range(steps):
            st = decoded[j]
            if st["status"] == -1:
                break
            force_ms = evs[2 * j].elapsed_time(evs[2 * j + 1])
            drv_ms = evs[2 * j + 1].elapsed_time(evs[2 * j + 2])
            _raise_for(st, self.step_index)
            flags = self.last_overlap_flags.copy() if self.collect_flags else None
            f_ms, m_ms, o_ms = _phase_ms(st["work"], force_ms if self._two_phase else 0.0, drv_ms,
                                         self._two_phase)
            res.append(StepStats(step=self.step_index, dt_used=st["dt_used"],
                                 overlap_iterations=st["overlap_iterations"], flip_passes=st["flip_passes"],
                                 inversion_repairs=st["inversion_repairs"], rollbacks=st["rollbacks"],
                                 n_overlapping=st["n_overlapping"], force_ms=f_ms, maintain_ms=m_ms,
                                 overlap_ms=o_ms, step_ms=force_ms + drv_ms, overlap_flags=flags,
                                 work=st["work"]))
            self.step_index += 1
        return res


def device_restore_delaunay(tri: PeriodicTriangulation, positions, box, tol=1e-12) -> int:
    """restore_delaunay (triangulation.py:319-334) on the GPU for a host position array."""
    torch = require_cuda()
    pos_np = np.ascontiguousarray(positions, dtype=np.float64)
    n = pos_np.shape[0]
    sys = ParticleSystem.__new__(ParticleSystem)
    dev = tri.device
    sys.box, sys.device = box, dev
    sys.positions_t = torch.from_numpy(pos_np).to(dev)
    sys.positions_prev_t = sys.positions_t.clone()
    sys.forces_t = torch.zeros_like(sys.positions_t)
    sys.alpha_t = torch.zeros(n, dtype=torch.float64, device=dev)
    sys.mu_t = torch.zeros(n, dtype=torch.float64, device=dev)
    sys.image_t = torch.zeros((n, 2), dtype=torch.int32, device=dev)
    params = SimParams(n=n, sigma=1.0, dt=0.01, diffusion=0.0)
    bp = make_params(params, box.length, 0, 0)
    bp.tol = float(tol)
    eng = _Engine(sys, tri, bp, 0)
    out = torch.zeros(1, dtype=torch.int64, device=dev)
    check(lib().bd_tri_restore_delaunay(ctypes.byref(eng.s), ctypes.byref(bp), ctypes.c_void_p(out.data_ptr()),
                                        _stream()), "bd_tri_restore_delaunay")
    passes = int(out.item())
    if passes < 0:
        raise NonConvergenceError("delaunay restoration did not converge")
    return passes


class LongRangeSimulation(_SimulationBase):
    """All-pairs forces with a continuously maintained triangulation
    (dynamics.py:177-274), every phase on the GPU; optionally the composite
    short-range / long+short force models (see module docstring)."""

    _two_phase = True

    def __init__(self, sys: ParticleSystem, params: SimParams, rng=None, tri: PeriodicTriangulation | None = None,
                 debug_scan: bool = False, collect_flags: bool = False, force: str = "long-range",
                 precision: str = "exact", skin: float | None = None, sharding=None):
        super().__init__(sys, params, rng, debug_scan, collect_flags)
        self.sharding = sharding  # distributed.ShardedLongRange: multi-GPU all-pairs
        if tri is None:
            from .triangulation import build_initial
            tri = build_initial(sys.positions, sys.box, device=sys.device)
        self.tri = tri
        if force not in FORCE_MODES:
            raise BrownsimError(f"unknown force model {force!r}; have {sorted(FORCE_MODES)}")
        if force != "long-range" and params.r_cutoff is None:
            raise BrownsimError("short-range force requires params.r_cutoff")
        if precision == "auto":  # EXACT for small systems; FAST-SYM while its partial buffer stays modest, else FAST
            import torch
            free, _ = torch.cuda.mem_get_info(sys.device)
            if sys.n <= AUTO_EXACT_MAX_N:
                precision = "exact"
            else:
                precision = "fast-sym" if lib().bd_long_range_workspace_bytes_for(sys.n, _abi.BD_LR_FAST_SYM) \
                    <= AUTO_SYM_FREE_FRACTION * free else "fast"
        if precision not in PRECISIONS:
            raise BrownsimError(f"unknown precision {precision!r}; have {sorted(PRECISIONS) + ['auto']}")
        self.force_model = force
        self.precision = precision
        self.skin = 0.5 * params.sigma if skin is None else float(skin)
        self.bparams = make_params(params, sys.box.length, self.rng.seed, self.rng.stream, FORCE_MODES[force],
                                   PRECISIONS[precision], skin, pairs=force != "long-range")
        self._eng = _Engine(sys, tri, self.bparams, self.rng.call)
        self._eng.clear_status()

    def _launch_force(self):
        if self.sharding is not None and self.sharding.world > 1:
            self.sharding.force(self._eng.s, self.bparams, _stream())
            return
        check(lib().bd_force(ctypes.byref(self._eng.s), ctypes.byref(self.bparams), _stream()), "bd_force")

    def _launch_driver(self, stats_ptr: int):
        check(lib().bd_maintain_tri(ctypes.byref(self._eng.s), ctypes.byref(self.bparams),
                                    ctypes.c_void_p(stats_ptr), _stream()), "bd_maintain_tri")


class ShortRangeSimulation(_SimulationBase):
    """Cutoff forces over Verlet lists; no triangulation (dynamics.py:307-346).

    The list covers max(r_cutoff, sigma) + skin and is rebuilt on the device
    once any particle moved more than skin/2 since the snapshot; overlap
    candidates are the pairs within sigma + skin at build time."""

    def __init__(self, sys: ParticleSystem, params: SimParams, rng=None, skin: float | None = None,
                 debug_scan: bool = False, collect_flags: bool = False):
        super().__init__(sys, params, rng, debug_scan, collect_flags)
        if params.r_cutoff is None:
            raise BrownsimError("short-range simulation requires r_cutoff")
        self.skin = 0.5 * params.sigma if skin is None else float(skin)
        self.r_list = max(params.r_cutoff, params.sigma) + self.skin
        self.overlap_margin = params.sigma + self.skin
        self.tri = None
        self.bparams = make_params(params, sys.box.length, self.rng.seed, self.rng.stream, _abi.BD_FORCE_SR,
                                   _abi.BD_LR_EXACT, self.skin, pairs=True)
        self._eng = _Engine(sys, None, self.bparams, self.rng.call)
        self._eng.clear_status()

    @property
    def verlet(self):
        """The current device Verlet list (pair_a, pair_b, snapshot) or None before the first step."""
        from .forces import VerletList
        meta = self._eng.vl_meta.cpu().numpy()
        if not meta[1]:
            return None
        k = int(meta[0])
        return VerletList(self._eng.pair_a[:k], self._eng.pair_b[:k], self._eng.vl_snap, self.r_list, self.skin)

    def _launch_driver(self, stats_ptr: int):
        check(lib().bd_step_verlet(ctypes.byref(self._eng.s), ctypes.byref(self.bparams),
                                   ctypes.c_void_p(stats_ptr), _stream()), "bd_step_verlet")


class AbpState(Versioned):
    """Director angles and self-propulsion parameters (dynamics.py:60-66).

    Once a simulation owns it, the angles live on the device (`angles_t`);
    the `angles` attribute reads them as a write-through numpy copy
    (`abp.angles[i] = v` reaches the device, like the reference's in-place
    numpy array)."""

    def __init__(self, angles, speed: float, rot_diffusion: float):
        self.speed = float(speed)
        self.rot_diffusion = float(rot_diffusion)
        self._host = np.ascontiguousarray(angles, dtype=np.float64).reshape(-1).copy()
        self.angles_t = None

    def bind(self, device):
        import torch
        if self.angles_t is None:
            self.angles_t = torch.from_numpy(self._host).to(device)
        return self.angles_t

    @property
    def angles(self) -> np.ndarray:
        return HostView(self.angles_t, self, "angles") if self.angles_t is not None else self._host

    @angles.setter
    def angles(self, value):
        import torch
        v = np.ascontiguousarray(value, dtype=np.float64).reshape(-1)
        if self.angles_t is not None:
            if v.shape != tuple(self.angles_t.shape):
                raise BrownsimError(f"angles must have shape {tuple(self.angles_t.shape)}, got {v.shape}")
            self.angles_t.copy_(torch.from_numpy(v))
            self.bump_version()
        else:
            self._host = v.copy()


class AbpSimulation(_SimulationBase):
    """Active Brownian particles (dynamics.py:349-399), one persistent kernel
    per step: Verlet list kept fresh, ballistic move by speed * dt along
    (cos theta, sin theta), angles += sqrt(2 D_r dt) xi (unclamped unless
    clamp_angle_noise), overlap rounds over the candidates within sigma + skin.

    The angular noise xi is the counter generator's normals(n) of one call
    per step (element i = pair i // 2, component i % 2)."""

    def __init__(self, sys: ParticleSystem, params: SimParams, rng, abp: AbpState, skin: float | None = None,
                 clamp_angle_noise: bool = False, debug_scan: bool = False, collect_flags: bool = False):
        super().__init__(sys, params, rng, debug_scan, collect_flags)
        self.abp = abp
        if abp.angles.shape != (sys.n,):
            raise BrownsimError(f"abp.angles must have shape ({sys.n},)")
        self.skin = 0.5 * params.sigma if skin is None else float(skin)
        self.r_list = params.sigma + self.skin
        self.overlap_margin = self.r_list
        self.clamp_angle_noise = bool(clamp_angle_noise)
        self.tri = None
        self.bparams = make_params(params, sys.box.length, self.rng.seed, self.rng.stream, _abi.BD_FORCE_SR,
                                   _abi.BD_LR_EXACT, self.skin, pairs=True, no_cutoff=True)
        self._refresh_params()
        self._eng = _Engine(sys, None, self.bparams, self.rng.call)
        self._eng.s.angles = abp.bind(sys.device).data_ptr()
        self._eng.clear_status()

    def _refresh_params(self):
        super()._refresh_params()
        self.bparams.abp_speed = float(self.abp.speed)
        self.bparams.abp_rot_diffusion = float(self.abp.rot_diffusion)
        self.bparams.abp_clamp_angle = int(self.clamp_angle_noise)

    verlet = ShortRangeSimulation.verlet

    def _launch_driver(self, stats_ptr: int):
        check(lib().bd_step_abp(ctypes.byref(self._eng.s), ctypes.byref(self.bparams),
                                ctypes.c_void_p(stats_ptr), _stream()), "bd_step_abp")
