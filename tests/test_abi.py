"""CPU: the C-ABI library builds, loads and exports every symbol declared in
include/kreg_b200.h; without a CUDA device the engine refuses to run (no CPU
fallback). Host-side pieces that need no device (SE(3), anneal_step,
check_config) are compared with the oracle."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

from paper_2012_03683_b200 import api, synth
from paper_2012_03683_b200.types import Isometry, RegistrationConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "kreg_b200.h")).read()
    return sorted(set(re.findall(r"\b(kreg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = api.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert L.kreg_abi_version() == 1


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    h = C.c_void_p()
    rc = api.lib().kreg_ctx_create(0, C.byref(h))
    assert rc == 6  # KREG_NO_DEVICE
    assert b"no CUDA device" in api.lib().kreg_last_error()


def test_host_se3_matches_oracle(oracle):
    rng = synth.SplitMix64(8001)
    for _ in range(200):
        xi = synth.random_twist(rng, 3.0, 5.0)
        a = api.se3_exp(xi)
        b = oracle.exp(xi)
        assert np.array_equal(a.as12(), b.as12())
        T = synth.random_isometry(rng, 1.0, 2.0)
        assert np.array_equal(api.se3_compose(a, T).as12(), oracle.compose(b, T).as12())
    # branch continuity at the Taylor switch (acceptance.cpp:318-327)
    axis = np.array([0.3, -0.5, 0.8]) / np.linalg.norm([0.3, -0.5, 0.8])
    lo = api.se3_exp(np.concatenate([axis * 1e-8 * (1 - 1e-9), [1, 2, 3]]))
    hi = api.se3_exp(np.concatenate([axis * 1e-8 * (1 + 1e-9), [1, 2, 3]]))
    assert np.abs(lo.as12() - hi.as12()).max() <= 1e-12
    with pytest.raises(ValueError):
        api.se3_exp([math.nan, 0, 0, 0, 0, 0])


def test_host_anneal_and_config_match_oracle(oracle):
    cfg = RegistrationConfig(stabilization_window=5, stabilization_rel_tol=1e-5, min_lengthscale=0.01)
    rng = np.random.default_rng(0)
    for _ in range(100):
        h = list(0.7 + 1e-6 * rng.standard_normal(rng.integers(1, 12)))
        l = float(rng.uniform(0.01, 0.5))
        assert api.anneal_step(l, h, cfg) == oracle.anneal_step(l, h, cfg)
    api.check_config(RegistrationConfig())
    for bad in (dict(decay_factor=1.5), dict(min_lengthscale=2.0), dict(max_iterations=0), dict(c_min=1.0),
                dict(step_shrink=1.0), dict(cutoff_multiplier=0.5)):
        with pytest.raises(ValueError):
            api.check_config(RegistrationConfig(**bad))


def test_diameter_matches_oracle(oracle):
    for n in (1, 50, 2500):
        X = synth.make_box_cloud(n, n)
        assert api.lib().kreg_cloud_diameter(X.view()) == oracle.diameter(X)
