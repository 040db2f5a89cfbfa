"""CPU: pin the plain-C oracle (oracle/kreg_oracle.c) against the golden
vectors made by the compiled reference, and — where the reference library is
built — against the reference directly. Mirrors the reference's own
hot-path tests (tests/test_inner_product.cpp, test_registration.cpp,
test_kernels.cpp, test_se3.cpp)."""
import math
import os

import numpy as np
import pytest

from paper_2012_03683_b200 import synth
from paper_2012_03683_b200.types import (Channel, ChannelKind, ChannelParams, FeatureSchema, Isometry, KernelForm,
                                         KernelParams, PointCloud, RegistrationConfig, compose, inverse,
                                         rotation_angle, translation_norm)

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_cloud(z, prefix, schema):
    return PointCloud(z[f"{prefix}_xyz"], schema, z[f"{prefix}_feat"] if schema.total_dim else None)


def load_params(z):
    return KernelParams(float(z["sigma"]), float(z["lengthscale"]),
                        [ChannelParams(a, b, KernelForm(int(c))) for a, b, c in z["per_channel"]])


COLOR = FeatureSchema([Channel("color", 3, ChannelKind.color)])


@pytest.mark.parametrize("seed", [101, 102, 103])
def test_generator_replicas_are_bit_exact(seed):
    z = np.load(os.path.join(GOLD, f"labeled_{seed}.npz"))
    X = synth.random_labeled_cloud(seed, 500, 1.0, True)
    assert np.array_equal(X.positions, z["X_xyz"]) and np.array_equal(X.features, z["X_feat"])
    rng = synth.SplitMix64(seed)
    T = synth.random_isometry(rng, 0.3, 0.2)
    assert np.allclose(T.as12(), z["T"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("seed", [101, 102, 103])
def test_oracle_pairs_match_golden_exactly(oracle, seed):
    # test_inner_product.cpp:90-105: grid pairs == brute force, bitwise
    z = np.load(os.path.join(GOLD, f"labeled_{seed}.npz"))
    X, Z = load_cloud(z, "X", COLOR), load_cloud(z, "Z", COLOR)
    p = load_params(z)
    for dense in (False, True):
        pr = oracle.build_pairs(X, Z, z["T"], p, 3.0, 1e-4, dense=dense)
        assert np.array_equal(pr.offsets, z["offsets"])
        assert np.array_equal(pr.x_index, z["x_index"])
        np.testing.assert_allclose(pr.coeff, z["coeff"], rtol=1e-14, atol=0)
    ev = oracle.objective_and_gradient(pr, X, Z, z["T"], p)
    np.testing.assert_allclose(ev, z["eval"], rtol=1e-12, atol=1e-12 * np.abs(z["eval"]).max())


def test_oracle_kitti_small_matches_golden(oracle):
    z = np.load(os.path.join(GOLD, "kitti_small.npz"))
    X, Z = load_cloud(z, "X", synth.KITTI_SCHEMA), load_cloud(z, "Z", synth.KITTI_SCHEMA)
    p = synth.kitti_params()
    k = 0
    for l in (0.1, 0.0475):
        pl = p.with_lengthscale(l)
        for T in z["Tlist"]:
            pr = oracle.build_pairs(X, Z, T, pl, 3.0, 1e-4)
            assert pr.size() == z["counts"][k]
            ev = oracle.objective_and_gradient(pr, X, Z, T, pl)
            np.testing.assert_allclose(ev, z["evals"][k], rtol=1e-11, atol=1e-11 * np.abs(z["evals"][k]).max())
            k += 1
    pr = oracle.build_pairs(X, Z, z["init"], p.with_lengthscale(0.1), 3.0, 1e-4)
    assert np.array_equal(pr.offsets, z["offsets"]) and np.array_equal(pr.x_index, z["x_index"])


def test_oracle_registration_matches_golden_box(oracle):
    z = np.load(os.path.join(GOLD, "box_registration.npz"))
    X, Z = PointCloud(z["X_xyz"]), PointCloud(z["Z_xyz"])
    cfg = RegistrationConfig(init_lengthscale=0.12, min_lengthscale=0.08, subsequent_lengthscale=0.12,
                             stabilization_window=3, max_iterations=600)
    res = oracle.register_clouds(X, Z, Isometry(), KernelParams(), cfg)
    assert res.iterations == int(z["reg_iterations"])
    assert res.converged == bool(z["reg_converged"])
    np.testing.assert_allclose(res.objective_trace, z["reg_objective"], rtol=1e-9)
    assert np.array_equal(res.lengthscale_trace, z["reg_lengthscale"])
    np.testing.assert_allclose(res.transform.as12(), z["reg_T"], atol=1e-9)
    err = compose(inverse(res.transform), Isometry.from12(z["T_star"]))
    assert rotation_angle(err) <= 0.5 * math.pi / 180.0


def test_oracle_kernel_known_answers(oracle):
    # test_kernels.cpp:10-21, test_inner_product.cpp:49-58
    one = PointCloud([[0.5, 0.5, 0.5]])
    p = KernelParams(lengthscale=0.1)
    pr = oracle.build_pairs(one, one, Isometry(), p, 3.0, 1e-4)
    assert pr.size() == 1 and pr.x_index[0] == 0 and pr.coeff[0] == 1.0
    a, b = PointCloud([[0, 0, 0]]), PointCloud([[0.5, 0, 0]])
    p = KernelParams(lengthscale=0.5)
    pr = oracle.build_pairs(a, b, Isometry(), p, 3.0, 0.0)
    assert oracle.inner_product(pr, a, b, Isometry(), p) == pytest.approx(0.6065306597126334, rel=1e-12)
    c = PointCloud([[1.5, 0, 0]])
    pr = oracle.build_pairs(a, c, Isometry(), p, 3.0, 0.0)
    assert oracle.inner_product(pr, a, c, Isometry(), p) == pytest.approx(0.011108996538242306, rel=1e-12)
    # orthogonal one-hot semantics are dropped (test_kernels.cpp:126-135)
    sch = FeatureSchema([Channel("sem", 3, ChannelKind.semantic)])
    u = PointCloud([[0, 0, 0]], sch, [[1.0, 0, 0]])
    v = PointCloud([[0, 0, 0]], sch, [[0, 1.0, 0]])
    pl = KernelParams(lengthscale=0.5, per_channel=[ChannelParams(1.0, 1.0, KernelForm.linear)])
    assert oracle.build_pairs(u, v, Isometry(), pl, 3.0, 1e-9).size() == 0


def test_oracle_fd_gradient(oracle):
    # test_inner_product.cpp:191-209 (left perturbation, central differences)
    rng = synth.SplitMix64(19)
    for inst in range(5):
        X = synth.random_labeled_cloud(1000 + inst, 50, 1.0, True, 3)
        Z = synth.random_labeled_cloud(2000 + inst, 50, 1.0, True, 3)
        T = synth.random_isometry(rng, 0.5, 0.3)
        p = synth.params_for(X, 0.25, 0.35)
        pr = oracle.build_pairs(X, Z, T, p, 1000.0, 0.0)
        g = oracle.objective_and_gradient(pr, X, Z, T, p)[1:]
        for k in range(6):
            d = np.zeros(6)
            d[k] = 1e-6
            fp = oracle.inner_product(pr, X, Z, oracle.compose(oracle.exp(d), T), p)
            fm = oracle.inner_product(pr, X, Z, oracle.compose(oracle.exp(-d), T), p)
            fd = (fp - fm) / 2e-6
            assert abs(g[k] - fd) <= 1e-5 * max(abs(fd), 1e-10) + 1e-10


def test_oracle_anneal_step(oracle):
    # test_registration.cpp:49-73
    cfg = RegistrationConfig(stabilization_window=5, stabilization_rel_tol=1e-5, min_lengthscale=0.01)
    assert oracle.anneal_step(0.5, [0.73] * 8, cfg) == 0.5 * 0.98
    assert oracle.anneal_step(0.5, [0.73] * 4, cfg) == 0.5
    assert oracle.anneal_step(0.5, [0.7, 0.8, 0.7, 0.8, 0.7, 0.8], cfg) == 0.5
    assert oracle.anneal_step(0.01, [0.73] * 8, cfg) == 0.01
    assert oracle.anneal_step(0.0101, [0.73] * 8, cfg) == 0.0101


def test_oracle_se3_exp_against_known_screw(oracle):
    # test_se3.cpp:27-40: pi/2 about z with v = (1,0,0) -> t = (2/pi, 2/pi, 0)
    T = oracle.exp([0, 0, math.pi / 2, 1, 0, 0])
    np.testing.assert_allclose(T.translation, [2 / math.pi, 2 / math.pi, 0], atol=1e-12)


# --------------------------------------------- against the compiled reference
def test_oracle_equals_reference_on_random_fixtures(oracle, ref):
    rng = synth.SplitMix64(43)
    for inst in range(3):
        X = synth.random_labeled_cloud(41 + inst, 300, 1.0, True, 4)
        Z = synth.random_labeled_cloud(42 + inst, 300, 1.0, True, 4)
        T = synth.random_isometry(rng, 0.2, 0.1)
        p = synth.params_for(X, 0.12, 0.3)
        a = oracle.build_pairs(X, Z, T, p, 3.0, 1e-4)
        b = ref.build_pairs(X, Z, T, p, 3.0, 1e-4)
        assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.x_index, b.x_index)
        np.testing.assert_allclose(a.coeff, b.coeff, rtol=1e-14)
        np.testing.assert_allclose(oracle.objective_and_gradient(a, X, Z, T, p),
                                   ref.objective_and_gradient(b, X, Z, T, p), rtol=1e-11, atol=1e-11)
        assert oracle.max_point_displacement(Z, T, Isometry()) == pytest.approx(
            ref.max_point_displacement(Z, T, Isometry()), rel=1e-15)


def test_oracle_registration_equals_reference(oracle, ref):
    X = synth.make_box_cloud(31, 400, False)
    rng = synth.SplitMix64(32)
    gt = synth.random_twist(rng, 8.0 * math.pi / 180.0, 0.04)
    Z = PointCloud(inverse(synth.se3_exp(gt)).apply(X.positions))
    cfg = RegistrationConfig(init_lengthscale=0.15, min_lengthscale=0.06, subsequent_lengthscale=0.15,
                             stabilization_window=3, max_iterations=600)
    a = oracle.register_clouds(X, Z, Isometry(), KernelParams(), cfg)
    b = ref.register_clouds(X, Z, Isometry(), KernelParams(), cfg)
    assert a.iterations == b.iterations and a.converged == b.converged
    assert np.array_equal(a.lengthscale_trace, b.lengthscale_trace)
    np.testing.assert_allclose(a.objective_trace, b.objective_trace, rtol=1e-9)
    np.testing.assert_allclose(a.transform.as12(), b.transform.as12(), atol=1e-9)


def test_generator_replicas_match_reference_helpers(ref):
    """synth.py replicas == tests/test_helpers.hpp compiled by GCC (incl. its
    right-to-left evaluation of Vector3d(f(), f(), f()) arguments)."""
    import ctypes as C
    from paper_2012_03683_b200 import _abi
    L = ref.lib
    L.kref_random_twists.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int, _abi.dptr]
    out = np.zeros((5, 6))
    L.kref_random_twists(19, 0.5, 0.3, 5, _abi.as_ptr(out))
    rng = synth.SplitMix64(19)
    assert np.array_equal(out, np.stack([synth.random_twist(rng, 0.5, 0.3) for _ in range(5)]))
    L.kref_random_labeled_cloud.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_int, C.c_int, _abi.dptr, _abi.dptr]
    xyz, f = np.zeros((50, 3)), np.zeros((50, 7))
    L.kref_random_labeled_cloud(101, 50, 1.0, 1, 4, _abi.as_ptr(xyz), _abi.as_ptr(f))
    c = synth.random_labeled_cloud(101, 50, 1.0, True, 4)
    assert np.array_equal(xyz, c.positions) and np.array_equal(f, c.features)
    L.kref_clustered_cloud.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, _abi.dptr,
                                       _abi.dptr]
    xyz, f = np.zeros((60, 3)), np.zeros((60, 3))
    L.kref_clustered_cloud(11, 3, 20, 5.0, 0.1, 1, _abi.as_ptr(xyz), _abi.as_ptr(f))
    c = synth.clustered_cloud(11, 3, 20, 5.0, 0.1, True)
    assert np.array_equal(xyz, c.positions) and np.array_equal(f, c.features)


def test_reference_builds_and_generators(ref):
    X = ref.make_box_cloud(7, 100, True)
    Y = synth.make_box_cloud(7, 100, True)
    assert np.array_equal(X.positions, Y.positions) and np.array_equal(X.features, Y.features)
    R = ref.make_ring_cloud(55, 8, 30, True)
    S = synth.make_ring_cloud(55, 8, 30, True)
    np.testing.assert_allclose(R.positions, S.positions, rtol=0, atol=1e-15)
