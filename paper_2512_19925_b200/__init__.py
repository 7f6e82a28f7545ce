"""hwwg — B200-native engine for the hybrid weight-window time-dependent Monte
Carlo history loop (arxiv 2512.19925).

The compute path is libhwwg.so (sm_100a CUDA + C++ host, C ABI in
include/hwwg.h); this package is the thin Python mirror of the reference's API.
"""
from ._capi import PARTICLE_DT, RNG_EXACT, RNG_PHILOX, HwwgError, LIB_PATH  # noqa: F401
from .hww import (  # noqa: F401
    Driver, Engine, Loopback, Material, Mesh1D, RunConfig, StepContext, StepOutcome, TallySet,
    WeightWindowGrid, build_uniform_mesh, default_engine, run, run_segment_parallel,
    ReferenceSolution, load_reference, save_reference, step_metrics, gauss_legendre, sn_solve,
    compute_reference)

__all__ = [
    "Driver", "Engine", "Loopback", "Material", "Mesh1D", "RunConfig", "StepContext", "StepOutcome",
    "TallySet", "WeightWindowGrid", "build_uniform_mesh", "default_engine", "run",
    "run_segment_parallel", "ReferenceSolution", "load_reference", "save_reference",
    "step_metrics", "gauss_legendre", "sn_solve", "compute_reference", "PARTICLE_DT", "RNG_EXACT", "RNG_PHILOX", "HwwgError", "LIB_PATH"]
