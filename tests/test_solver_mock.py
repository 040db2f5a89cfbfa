"""CPU: the product's host solver (csrc/solver.cpp) driven by the C oracle in
place of the device (tests/native/mock_round.cpp) must reproduce the
reference registration loop's decisions and traces exactly — including with
K-candidate batching, gradient reuse and memoisation switched on."""
import ctypes as C
import math
import os
import subprocess

import numpy as np
import pytest

from paper_2012_03683_b200 import _abi, synth
from paper_2012_03683_b200.types import (Isometry, KernelParams, PointCloud, RegistrationConfig, RegistrationResult,
                                         inverse)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "native", "libmock_solver.so")


@pytest.fixture(scope="module")
def mock():
    subprocess.check_call(["make", "-s", "-C", os.path.join(HERE, "native")], stderr=subprocess.DEVNULL)
    L = C.CDLL(LIB)
    L.mock_register.argtypes = [C.POINTER(_abi.kreg_cloud_view), C.POINTER(_abi.kreg_cloud_view), _abi.dptr,
                                C.POINTER(_abi.kreg_kernel_params), C.POINTER(_abi.kreg_registration_config),
                                C.POINTER(_abi.kreg_registration_result), C.c_int]
    return L


def run_mock(L, X, Z, init, params, cfg, k_first):
    buf = _abi.TraceBuffers(cfg.max_iterations)
    t = init.as12()
    c = cfg.cstruct()
    rc = L.mock_register(X.view(), Z.view(), _abi.as_ptr(t), params.cstruct(), C.byref(c), C.byref(buf.struct), k_first)
    return rc, RegistrationResult.from_buffers(buf)


def cases():
    X = synth.make_box_cloud(31, 300, False)
    rng = synth.SplitMix64(32)
    Z = PointCloud(inverse(synth.se3_exp(synth.random_twist(rng, 8.0 * math.pi / 180.0, 0.04))).apply(X.positions))
    yield X, Z, Isometry(), KernelParams(), RegistrationConfig(init_lengthscale=0.15, min_lengthscale=0.06,
                                                                  subsequent_lengthscale=0.15, stabilization_window=3,
                                                                  max_iterations=400)
    ring = synth.make_ring_cloud(55, 8, 20, True)
    Zr = PointCloud(inverse(synth.se3_exp([0, 0, 0.52, 0, 0, 0])).apply(ring.positions), ring.schema, ring.features)
    yield ring, Zr, Isometry(), synth.params_for(ring, 0.5, 0.2), RegistrationConfig(
        init_lengthscale=0.5, min_lengthscale=0.1, stabilization_window=3, max_iterations=400)
    Xk, Zk, Ts = synth.kitti_pair(11, 1500)
    yield Xk, Zk, synth.perturbed(Ts, 5), synth.kitti_params(), RegistrationConfig(
        init_lengthscale=0.3, min_lengthscale=0.2, stabilization_window=5, max_iterations=300)


@pytest.mark.parametrize("k_first", [1, 2, 3, 8])
def test_mock_solver_reproduces_reference_loop(mock, oracle, k_first):
    for X, Z, init, p, cfg in cases():
        want = oracle.register_clouds(X, Z, init, p, cfg)
        rc, got = run_mock(mock, X, Z, init, p, cfg, k_first)
        assert rc == 0
        assert got.iterations == want.iterations
        assert got.converged == want.converged
        assert np.array_equal(got.objective_trace, want.objective_trace)
        assert np.array_equal(got.lengthscale_trace, want.lengthscale_trace)
        assert np.array_equal(got.step_trace, want.step_trace)
        assert np.array_equal(got.twist_norm_trace, want.twist_norm_trace)
        assert np.array_equal(got.pair_count_trace, want.pair_count_trace)
        assert np.array_equal(got.rebuild_trace, want.rebuild_trace)
        assert np.array_equal(got.transform.as12(), want.transform.as12())


def test_mock_solver_no_overlap(mock):
    a, b = PointCloud([[0, 0, 0]]), PointCloud([[1000, 0, 0]])
    rc, _ = run_mock(mock, a, b, Isometry(), KernelParams(), RegistrationConfig(init_lengthscale=0.1,
                                                                                min_lengthscale=0.05), 2)
    assert rc == 2
