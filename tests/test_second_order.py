"""Second-order step-size terms (north_star item (4); a diagnostic with no
reference counterpart): {F, dF/d eps, d2F/d eps2} along
eps -> exp(eps xi) T with the pair list fixed.

CPU: the oracle restatement against central finite differences of the
oracle's inner_product (pins the formula). GPU: the fused sweep's extra
reductions against the oracle (1e-4 relative, the north_star tolerance) and
F' against the gradient's projection on xi."""
import numpy as np
import pytest

from paper_2012_03683_b200 import synth
from paper_2012_03683_b200.types import PointCloud, inverse


def _fd(oracle, pr, X, Z, T, xi, params, h):
    f = lambda e: oracle.inner_product(pr, X, Z, oracle.compose(oracle.exp(np.asarray(xi) * e), T), params)  # noqa: E731
    f0, fp, fm = f(0.0), f(h), f(-h)
    return f0, (fp - fm) / (2 * h), (fp - 2 * f0 + fm) / (h * h)


def _case(seed, n=3000):
    X, Z, T = synth.kitti_pair(seed, n)
    p = synth.kitti_params()
    rng = np.random.default_rng(seed)
    xi = rng.normal(size=6)
    xi /= np.linalg.norm(xi)
    return X, Z, synth.perturbed(T, seed), p, xi


@pytest.mark.parametrize("seed", [21, 22])
def test_oracle_terms_match_finite_differences(oracle, seed):
    X, Z, T, p, xi = _case(seed)
    pr = oracle.build_pairs(X, Z, T, p, 3.0, 1e-4)
    F, d1, d2 = oracle.directional_terms(pr, X, Z, T, xi, p)
    # Richardson-extrapolated central differences (O(h^4) truncation)
    f0, a1, a2 = _fd(oracle, pr, X, Z, T, xi, p, 2e-4)
    _, b1, b2 = _fd(oracle, pr, X, Z, T, xi, p, 1e-4)
    g1, g2 = (4 * b1 - a1) / 3, (4 * b2 - a2) / 3
    assert abs(F - f0) <= 1e-12 * abs(f0)
    assert abs(d1 - g1) <= 1e-6 * abs(g1)
    assert abs(d2 - g2) <= 1e-5 * abs(g2)


def test_oracle_first_derivative_is_gradient_projection(oracle):
    X, Z, T, p, xi = _case(23)
    pr = oracle.build_pairs(X, Z, T, p, 3.0, 1e-4)
    og = oracle.objective_and_gradient(pr, X, Z, T, p)
    _, d1, _ = oracle.directional_terms(pr, X, Z, T, xi, p)
    assert abs(d1 - og[1:] @ xi) <= 1e-10 * abs(d1)


@pytest.mark.gpu
@pytest.mark.parametrize("seed,n", [(21, 3000), (24, 40000)])
def test_device_terms_match_oracle(ctx, oracle, seed, n):
    from paper_2012_03683_b200 import api
    X, Z, T, p, xi = _case(seed, n)
    g = api.build_pairs(X, Z, T, p, 3.0, 1e-4, ctx=ctx)
    pr = oracle.build_pairs(X, Z, T, p, 3.0, 1e-4)
    dev = api.directional_terms(g, X, Z, T, xi, p)
    ref = oracle.directional_terms(pr, X, Z, T, xi, p)
    for k in range(3):
        assert abs(dev[k] - ref[k]) <= 1e-4 * max(abs(ref[k]), 1e-3 * abs(ref[0])), (k, dev, ref)
    # the first derivative is the device gradient projected on xi
    ev = api.objective_and_gradient(g, X, Z, T, p)
    assert abs(dev[1] - ev.grad @ xi) <= 1e-4 * max(abs(dev[1]), 1e-3 * abs(dev[0]))


@pytest.mark.gpu
def test_device_terms_geometric_box_and_newton_step(ctx, oracle):
    """Geometric-only box: near the optimum along the gradient direction the
    curvature is negative and the Newton step -F'/F'' is a positive step."""
    from paper_2012_03683_b200 import api
    from paper_2012_03683_b200.types import KernelParams, RegistrationConfig
    Xb = synth.make_box_cloud(2024, 2000, False)
    Tst = synth.se3_exp([0.01, -0.006, 0.008, 0.004, 0.002, -0.003])
    Zb = PointCloud(inverse(Tst).apply(Xb.positions))
    p = KernelParams(1.0, 0.1)
    from paper_2012_03683_b200.types import Isometry
    T = Isometry()
    g = api.build_pairs(Xb, Zb, T, p, 3.0, 1e-4, ctx=ctx)
    ev = api.objective_and_gradient(g, Xb, Zb, T, p)
    xi = ev.grad / np.linalg.norm(ev.grad)
    dev = api.directional_terms(g, Xb, Zb, T, xi, p)
    ref = oracle.directional_terms(oracle.build_pairs(Xb, Zb, T, p, 3.0, 1e-4), Xb, Zb, T, xi, p)
    assert np.allclose(dev, ref, rtol=1e-4)
    assert dev[1] > 0 and dev[2] < 0 and -dev[1] / dev[2] > 0
