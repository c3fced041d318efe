"""paper_1703_02484_b200 -- B200-native Brownian-dynamics hot path.

Drop-in for the per-timestep path of the reference package `brownsim`
(arXiv 1703.02484): same public names for setup, force models, step/run and
state read-out; every step runs on the GPU through libbd_b200.so
(hand-written sm_100a CUDA, include/bd_b200.h).  See DESIGN.md.
"""

from .core import (BrownsimError, BuildError, ConfigError, CounterRng, NonConvergenceError, ParticleSystem,
                   PeriodicBox, RngStream, SimParams, SingularityError, StepFailure, box_length_for_density,
                   clamped_gaussian, clamped_normals, min_image_disp, wrap)
from .initial import InitConfig, init_arrays, init_system, reservoir_sample, triangular_lattice

__version__ = "0.1.0"


def __getattr__(name):
    # GPU-side modules load lazily so that `import paper_1703_02484_b200` works
    # on a CPU-only host for setup / build tooling
    if name in ("LongRangeSimulation", "ShortRangeSimulation", "AbpSimulation", "AbpState", "StepStats",
                "MissedOverlapError", "integrate", "correct_overlaps"):
        from . import dynamics
        return getattr(dynamics, name)
    if name in ("PeriodicTriangulation", "build_initial", "incircle", "AuditReport", "RepairResult",
                "FlipDecision"):
        from . import triangulation
        return getattr(triangulation, name)
    raise AttributeError(name)
