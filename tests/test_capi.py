"""CPU checks of the product boundary: libhwwg.so loads, exports every symbol
include/hwwg.h declares, and its host logic (config defaults / loader /
validation) mirrors the reference. No compute calls: there is no GPU here."""
import ctypes as C
import os
import re

import pytest

import paper_2512_19925_b200 as hw
from paper_2512_19925_b200 import _capi as A

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "hwwg.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hwwg_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = A.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(A.EXPORTS)


def test_library_is_sm100a():
    data = open(A.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_default_config_matches_reference():
    c = A.RunConfigC()
    A.lib().hwwg_default_config(C.byref(c))
    # proj/include/hww/config.hpp:33-66
    assert (c.mode, c.histories_per_step, c.theta, c.rho, c.eps_min, c.u_ww) == (
        2, 10000, 0.5, 1.25, 1e-3, 3)
    assert list(c.fractions[:3]) == [0.25, 0.5, 0.75] and c.n_fractions == 3
    assert (c.ma_base_k, c.batches, c.seed, c.cells, c.time_steps) == (3, 20, 1, 201, 20)
    assert (c.sigma_t, c.sigma_f, c.nu_f, c.x_min, c.x_max) == (1.0, 1 / 3, 2.3, -20.5, 20.5)


def test_config_file_loader(tmp_path):
    p = tmp_path / "c.cfg"
    p.write_text("# comment\nmode = hww_ma\nhistories_per_step = 123  # trailing\n"
                 "update_fractions = 0.2, 0.4\nu_ww = 2\nsigma_s = 0.9\nsigma_f = 0\nrho=5\n")
    cfg = hw.RunConfig.from_file(p)
    assert cfg.mode == "hww_ma" and cfg.histories_per_step == 123 and cfg.rho == 5.0
    assert tuple(cfg.update_fractions) == (0.2, 0.4) and cfg.u_ww == 2
    assert cfg.material.sigma_s == 0.9 and cfg.material.sigma_f == 0.0
    assert cfg.validate() == []
    p.write_text("bogus = 1\n")
    with pytest.raises(ValueError, match="unknown key"):
        hw.RunConfig.from_file(p)
    p.write_text("mode = fancy\n")
    with pytest.raises(ValueError, match="unknown mode"):
        hw.RunConfig.from_file(p)
    p.write_text("just words\n")
    with pytest.raises(ValueError, match="expected key = value"):
        hw.RunConfig.from_file(p)


def test_config_file_loader_config3_keys(tmp_path):
    """The config-3 extension keys (regions, volumetric source, no pulse) load into
    the same RunConfig the BASELINE builder makes (paper_2512_19925_b200/configs.py)."""
    from paper_2512_19925_b200.configs import baseline
    p = tmp_path / "c3.cfg"
    p.write_text("mode = hww\nhistories_per_step = 10000000\nrho = 4\nseed = 3\n"
                 "x_min = 0\nx_max = 30\ncells = 1000\nt_end = 25\ntime_steps = 50\n"
                 "sigma_t = 1\nsigma_s = 0.5\nsigma_f = 0\nnu_f = 0\n"
                 "region = 10, 1, 0.5, 0, 0, 1\nregion = 20, 10, 1, 0, 0, 1\n"
                 "region = 30, 1, 0.99, 0, 0, 1\nvolume_source = 0, 2, 0, 1, 1\nno_pulse = 1\n")
    got, want = hw.RunConfig.from_file(p).to_c(), baseline(3).to_c()
    for f, _ in want._fields_:
        a, b = getattr(got, f), getattr(want, f)
        if hasattr(a, "__len__"):
            a, b = [list(x) if hasattr(x, "__len__") else x for x in a], \
                   [list(x) if hasattr(x, "__len__") else x for x in b]
        assert a == b, f
    p.write_text("region = 10, 1, 0.5\n")
    with pytest.raises(ValueError, match="region needs"):
        hw.RunConfig.from_file(p)


def test_config_validation_messages():
    cfg = hw.RunConfig(theta=0.3, rho=0.5, batches=1, update_fractions=(0.5, 0.25))
    v = cfg.validate()
    assert "theta must lie in [1/2, 1]" in v
    assert "rho must be >= 1" in v
    assert "batches must be >= 2" in v
    assert "update fractions must increase" in v


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(hw.HwwgError, match="no CUDA device"):
        hw.Engine()
    with pytest.raises(hw.HwwgError, match="no CUDA device"):
        hw.Driver(hw.RunConfig())
