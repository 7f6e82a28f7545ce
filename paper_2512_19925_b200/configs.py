"""The BASELINE.json configurations as RunConfigs (SURVEY.md §8(d) states the
choices the configs leave open: reference defaults for unspecified parameters,
seeds 3 (C3) and 1 (C4), C3's unit emission per unit time, C4's window mode
hww with the reference default rho = 1.25, C1's "filtered" = hww_ma k = 3).

    baseline(2)                        config 2 as stated
    baseline(5, rho=10.0, ma_base_k=2) one config-5 sweep point
    baseline(4, histories=12_500_000)  one GPU's share of config 4's 1e8 over 8
"""
from __future__ import annotations

from .hww import Material, RunConfig

# The config-5 sweep: window ratio x closure filter ("none" = hww, k = MA half-width).
C5_VARIANTS = [(rho, k) for rho in (2.0, 5.0, 10.0) for k in (0, 1, 2)]

DESCRIPTION = {
    1: "BASELINE config 1: slab [-20,20] 200 cells sigma_t=1 c=1 v=1, pulse x=0, 20 x dt=1, "
       "1e5 histories/step, hww_ma k=3 (filtered LOSM, reference default), rho=5, seed 42",
    2: "BASELINE config 2: slab [-20,20] 400 cells sigma_t=1 c=0.9 v=1, pulse x=0, 40 x dt=0.5, "
       "1e6 histories/step, hww_ma k=1, rho=5, seed 7",
    3: "BASELINE config 3: slab [0,30] 1000 cells, regions sigma_t=1/10/1 c=0.5/0.1/0.99, "
       "isotropic volumetric source x in [0,2] t in [0,1] (unit emission per unit time), "
       "50 x dt=0.5, 1e7 histories/step, hww rho=4, vacuum, seed 3",
    4: "BASELINE config 4: slab [-50,50] 4000 cells sigma_t=1 c=0.99 v=1, pulse x=0, "
       "100 x dt=0.5, 1e8 histories/step over 8 GPUs, hww rho=1.25 (reference defaults), seed 1",
    5: "BASELINE config 5: config-2 geometry (slab [-20,20] 400 cells c=0.9, 40 x dt=0.5), "
       "1e7 histories/step, seed 11, sweep rho in {2,5,10} x filter {none, MA3, MA5}",
}


def baseline(which: int, histories=None, time_steps=None, **kw) -> RunConfig:
    if which == 1:
        c = dict(mode="hww_ma", ma_base_k=3, histories_per_step=100_000, rho=5.0, seed=42,
                 material=Material(1.0, 1.0, 0.0, 0.0, 1.0), x_min=-20.0, x_max=20.0,
                 cells=200, t_end=20.0, time_steps=20)
    elif which == 2:
        c = dict(mode="hww_ma", ma_base_k=1, histories_per_step=1_000_000, rho=5.0, seed=7,
                 material=Material(1.0, 0.9, 0.0, 0.0, 1.0), x_min=-20.0, x_max=20.0,
                 cells=400, t_end=20.0, time_steps=40)
    elif which == 3:
        regions = [(10.0, Material(1.0, 0.5, 0.0, 0.0, 1.0)),
                   (20.0, Material(10.0, 1.0, 0.0, 0.0, 1.0)),
                   (30.0, Material(1.0, 0.99, 0.0, 0.0, 1.0))]
        c = dict(mode="hww", histories_per_step=10_000_000, rho=4.0, seed=3,
                 material=Material(1.0, 0.5, 0.0, 0.0, 1.0), x_min=0.0, x_max=30.0,
                 cells=1000, t_end=25.0, time_steps=50, regions=regions,
                 volume_source=(0.0, 2.0, 0.0, 1.0, 1.0), no_pulse=True)
    elif which == 4:
        c = dict(mode="hww", histories_per_step=100_000_000, rho=1.25, seed=1,
                 material=Material(1.0, 0.99, 0.0, 0.0, 1.0), x_min=-50.0, x_max=50.0,
                 cells=4000, t_end=50.0, time_steps=100)
    elif which == 5:
        c = dict(mode="hww_ma", ma_base_k=1, histories_per_step=10_000_000, rho=5.0, seed=11,
                 material=Material(1.0, 0.9, 0.0, 0.0, 1.0), x_min=-20.0, x_max=20.0,
                 cells=400, t_end=20.0, time_steps=40)
    elif which == 0:  # the reference's own proj/configs/benchmark.cfg (the fission case)
        c = dict(mode="hww", ma_base_k=3, histories_per_step=10_000, rho=1.25, seed=1,
                 material=Material(1.0, 1.0 / 3.0, 1.0 / 3.0, 2.3, 1.0), x_min=-20.5,
                 x_max=20.5, cells=201, t_end=20.0, time_steps=20)
    else:
        raise ValueError(which)
    if which == 5 and kw.get("ma_base_k", 1) == 0:  # "none": the unfiltered hww mode
        kw = dict(kw)
        kw.pop("ma_base_k")
        kw["mode"] = "hww"
    c.update(kw)
    if histories is not None:
        c["histories_per_step"] = histories
    if time_steps is not None:
        dt = c["t_end"] / c["time_steps"]
        c["time_steps"], c["t_end"] = time_steps, dt * time_steps
    return RunConfig(**c)
