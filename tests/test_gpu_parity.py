"""GPU parity tests: the CUDA path through the C-ABI (libkreg_b200.so) against
the golden vectors made by the compiled reference, the compiled reference
itself (oracle/_ref) and the plain-C oracle. Tolerances are those of
BASELINE.json:north_star:
  * neighbour sets identical except pairs within 1e-6 m of the cutoff (plus
    |c - c_min| <= 1e-5 c_min: c is computed in FP32 on the device);
  * per-evaluation F and grad within 1e-4 relative (grad: vector norm);
  * final rotation / translation within 1e-3 rad / 1e-3 m.
"""
import math
import os

import numpy as np
import pytest

from paper_2012_03683_b200 import api, synth
from paper_2012_03683_b200.types import (Channel, ChannelKind, ChannelParams, FeatureSchema, Isometry, KernelForm,
                                         KernelParams, NoOverlapError, PointCloud, RegistrationConfig, compose,
                                         inverse, rotation_angle, translation_norm)

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
COLOR = FeatureSchema([Channel("color", 3, ChannelKind.color)])


def load_cloud(z, prefix, schema):
    return PointCloud(z[f"{prefix}_xyz"], schema, z[f"{prefix}_feat"] if schema.total_dim else None)


def load_params(z):
    return KernelParams(float(z["sigma"]), float(z["lengthscale"]),
                        [ChannelParams(a, b, KernelForm(int(c))) for a, b, c in z["per_channel"]])


def assert_eval_close(got, want, rtol=1e-4):
    got, want = np.asarray(got, dtype=float), np.asarray(want, dtype=float)
    assert abs(got[0] - want[0]) <= rtol * abs(want[0]) + 1e-12, (got[0], want[0])
    gw, ww = got[1:7], want[1:7]
    assert np.linalg.norm(gw - ww) <= rtol * np.linalg.norm(ww) + 1e-12, (gw, ww)


def feature_coefficient(u, v, schema, params):
    """kernels.cpp:18-53 in float64 (for tie classification only)."""
    c, off = 1.0, 0
    for ch, cp in zip(schema.channels, params.per_channel):
        a, b = u[off:off + ch.dim], v[off:off + ch.dim]
        if cp.form == KernelForm.linear:
            c *= float(np.dot(a, b))
        else:
            c *= cp.sigma ** 2 * math.exp(-float(np.sum((a - b) ** 2)) / (2 * cp.lengthscale ** 2))
        off += ch.dim
    return c


def assert_pairs_match(got, want, X, Z, T, params, cutoff_mult, c_min):
    """Pair sets identical except boundary ties (north_star tolerance)."""
    off_g, idx_g, cf_g = got
    off_w, idx_w, cf_w = want
    T = T if isinstance(T, Isometry) else Isometry.from12(T)
    q = T.apply(Z.positions)
    cutoff = cutoff_mult * params.lengthscale
    n_tie = 0
    for j in range(Z.size()):
        g = dict(zip(idx_g[off_g[j]:off_g[j + 1]].tolist(), cf_g[off_g[j]:off_g[j + 1]].tolist()))
        w = dict(zip(idx_w[off_w[j]:off_w[j + 1]].tolist(), cf_w[off_w[j]:off_w[j + 1]].tolist()))
        for i in set(g) ^ set(w):
            d = float(np.linalg.norm(X.positions[i] - q[j]))
            c = feature_coefficient(X.features[i], Z.features[j], X.schema, params) if X.schema.total_dim else 1.0
            assert abs(d - cutoff) <= 1e-6 or abs(c - c_min) <= 1e-5 * max(c_min, 1e-300), (j, i, d, cutoff, c)
            n_tie += 1
        for i in set(g) & set(w):
            assert abs(g[i] - w[i]) <= 1e-5 * abs(w[i]) + 1e-12, (j, i, g[i], w[i])
        # reference order inside a group: ascending i
        assert list(idx_g[off_g[j]:off_g[j + 1]]) == sorted(idx_g[off_g[j]:off_g[j + 1]])
    assert n_tie <= max(2, len(idx_w) // 10000)


# ----------------------------------------------------------- golden vectors
@pytest.mark.parametrize("seed", [101, 102, 103])
def test_pairs_and_eval_match_golden(ctx, seed):
    z = np.load(os.path.join(GOLD, f"labeled_{seed}.npz"))
    X, Z = load_cloud(z, "X", COLOR), load_cloud(z, "Z", COLOR)
    p = load_params(z)
    pr = api.build_pairs(X, Z, z["T"], p, 3.0, 1e-4)
    assert pr.size() == len(z["x_index"]) or abs(pr.size() - len(z["x_index"])) <= 2
    assert_pairs_match(pr.export(), (z["offsets"], z["x_index"], z["coeff"]), X, Z, z["T"], p, 3.0, 1e-4)
    ev = api.objective_and_gradient(pr, X, Z, z["T"], p)
    assert_eval_close([ev.value, *ev.grad], z["eval"])


def test_kitti_small_matches_golden(ctx):
    z = np.load(os.path.join(GOLD, "kitti_small.npz"))
    X, Z = load_cloud(z, "X", synth.KITTI_SCHEMA), load_cloud(z, "Z", synth.KITTI_SCHEMA)
    p = synth.kitti_params()
    k = 0
    for l in (0.1, 0.0475):
        pl = p.with_lengthscale(l)
        for T in z["Tlist"]:
            pr = api.build_pairs(X, Z, T, pl, 3.0, 1e-4)
            assert abs(pr.size() - int(z["counts"][k])) <= 2
            ev = api.objective_and_gradient(pr, X, Z, T, pl)
            assert_eval_close([ev.value, *ev.grad], z["evals"][k])
            k += 1
    pr = api.build_pairs(X, Z, z["init"], p.with_lengthscale(0.1), 3.0, 1e-4)
    assert_pairs_match(pr.export(), (z["offsets"], z["x_index"], z["coeff"]), X, Z, z["init"],
                       p.with_lengthscale(0.1), 3.0, 1e-4)


def test_box_registration_matches_golden(ctx):
    z = np.load(os.path.join(GOLD, "box_registration.npz"))
    X, Z = PointCloud(z["X_xyz"]), PointCloud(z["Z_xyz"])
    cfg = RegistrationConfig(init_lengthscale=0.12, min_lengthscale=0.08, subsequent_lengthscale=0.12,
                             stabilization_window=3, max_iterations=600)
    res = api.register_clouds(X, Z, Isometry(), KernelParams(), cfg)
    ref_T = Isometry.from12(z["reg_T"])
    err = compose(inverse(res.transform), ref_T)
    assert rotation_angle(err) <= 1e-3 and translation_norm(err) <= 1e-3
    assert res.converged
    # the traces obey the reference's invariants
    ls = res.lengthscale_trace
    for a, b in zip(ls[:-1], ls[1:]):
        assert b == a or b == a * 0.98
    truth = compose(inverse(res.transform), Isometry.from12(z["T_star"]))
    assert rotation_angle(truth) <= 0.5 * math.pi / 180


def test_kitti_small_registration_matches_golden(ctx):
    z = np.load(os.path.join(GOLD, "kitti_small.npz"))
    X, Z = load_cloud(z, "X", synth.KITTI_SCHEMA), load_cloud(z, "Z", synth.KITTI_SCHEMA)
    res = api.register_clouds(X, Z, z["init"], synth.kitti_params(), synth.kitti_subsequent_config())
    err = compose(inverse(res.transform), Isometry.from12(z["reg_T"]))
    assert rotation_angle(err) <= 1e-3 and translation_norm(err) <= 1e-3, (rotation_angle(err), translation_norm(err))
    assert res.converged == bool(z["reg_converged"])


# ------------------------------------------------------ against the reference
def test_kitti_full_size_pairs_and_eval_vs_reference(ctx, ref):
    X, Z, Ts = synth.kitti_pair(7, 40000)
    p = synth.kitti_params()
    init = synth.perturbed(Ts, 3)
    for l in (0.1, 0.0475):
        pl = p.with_lengthscale(l)
        g = api.build_pairs(X, Z, init, pl, 3.0, 1e-4)
        r = ref.build_pairs(X, Z, init, pl, 3.0, 1e-4)
        assert abs(g.size() - r.size()) <= 2
        assert_pairs_match(g.export(), (r.offsets, r.x_index, r.coeff), X, Z, init, pl, 3.0, 1e-4)
        for T in (init, Ts, synth.perturbed(Ts, 4, 0.01, 0.1)):
            ev = api.objective_and_gradient(g, X, Z, T, pl)
            assert_eval_close([ev.value, *ev.grad], ref.objective_and_gradient(r, X, Z, T, pl))


def test_candidate_list_rebuild_is_exact(ctx, ref):
    """A rebuild that filters the resident candidate list (R_s = cutoff (1 +
    skin) around the earlier transform) yields exactly the list a grid search
    at the new transform yields, and the reference's set."""
    X, Z, Ts = synth.kitti_pair(7, 40000)
    p = synth.kitti_params()
    init = synth.perturbed(Ts, 3)
    c = api.default_context()
    c.reset_stats()
    g = api.build_pairs(X, Z, init, p, 3.0, 1e-4)
    first = c.build_stats()  # (a capacity overflow re-runs the grid search)
    assert first["grid_builds"] >= 1 and first["filter_builds"] == 0
    rng = synth.SplitMix64(11)
    T1 = compose(synth.random_isometry(rng, math.radians(0.05), 0.01), init)  # moves < R_s - cutoff
    p1 = p.with_lengthscale(0.098)
    g.rebuild(T1, p1, 3.0, 1e-4)
    st = c.build_stats()
    assert st["grid_builds"] == first["grid_builds"] and st["filter_builds"] >= 1
    fresh = api.build_pairs(X, Z, T1, p1, 3.0, 1e-4)
    a, b = g.export(), fresh.export()
    # both lists apply the cutoff in FP32 from different candidate origins:
    # identical up to pairs within the 1e-6 m tie band
    assert abs(g.size() - fresh.size()) <= 2
    assert_pairs_match(a, b, X, Z, T1, p1, 3.0, 1e-4)
    r = ref.build_pairs(X, Z, T1, p1, 3.0, 1e-4)
    assert_pairs_match(a, (r.offsets, r.x_index, r.coeff), X, Z, T1, p1, 3.0, 1e-4)
    ev_g = api.objective_and_gradient(g, X, Z, T1, p1)
    assert_eval_close([ev_g.value, *ev_g.grad], ref.objective_and_gradient(r, X, Z, T1, p1))
    # a move beyond the skin falls back to a grid search
    T2 = compose(synth.random_isometry(rng, math.radians(2.0), 0.5), T1)
    before = c.build_stats()
    g.rebuild(T2, p1, 3.0, 1e-4)
    assert c.build_stats()["grid_builds"] == before["grid_builds"] + 1
    fresh2 = api.build_pairs(X, Z, T2, p1, 3.0, 1e-4)
    assert_pairs_match(g.export(), fresh2.export(), X, Z, T2, p1, 3.0, 1e-4)


def test_tum_shaped_eval_vs_reference(ctx, ref):
    X, Z, Ts = synth.tum_pair(3, 20000)
    p = synth.tum_params()
    g = api.build_pairs(X, Z, Ts, p, 3.0, 1e-4)
    r = ref.build_pairs(X, Z, Ts, p, 3.0, 1e-4)
    assert abs(g.size() - r.size()) <= 2
    ev = api.objective_and_gradient(g, X, Z, Ts, p)
    assert_eval_close([ev.value, *ev.grad], ref.objective_and_gradient(r, X, Z, Ts, p))


def test_geometric_box_5k_vs_reference(ctx, ref):
    X = synth.make_box_cloud(2012036830, 5000, False)
    rng = synth.SplitMix64(5)
    T = synth.random_isometry(rng, 0.1, 0.05)
    p = KernelParams(lengthscale=0.1)
    g = api.build_pairs(X, X, T, p, 3.0, 1e-4)
    r = ref.build_pairs(X, X, T, p, 3.0, 1e-4)
    assert abs(g.size() - r.size()) <= 2
    ev = api.objective_and_gradient(g, X, X, T, p)
    assert_eval_close([ev.value, *ev.grad], ref.objective_and_gradient(r, X, X, T, p))
    assert api.max_point_displacement(X, T, Isometry()) == pytest.approx(
        ref.max_point_displacement(X, T, Isometry()), rel=1e-12)


def test_fd_gradient_of_gpu_value(ctx, oracle):
    # test_inner_product.cpp:191-209 on the device value
    rng = synth.SplitMix64(19)
    for inst in range(4):
        X = synth.random_labeled_cloud(1000 + inst, 50, 1.0, True, 3)
        Z = synth.random_labeled_cloud(2000 + inst, 50, 1.0, True, 3)
        T = synth.random_isometry(rng, 0.5, 0.3)
        p = synth.params_for(X, 0.25, 0.35)
        pr = oracle.build_pairs(X, Z, T, p, 1000.0, 0.0)
        g = api.build_pairs(X, Z, T, p, 1000.0, 0.0)
        ev = api.objective_and_gradient(g, X, Z, T, p)
        fd = np.zeros(6)
        for k in range(6):
            d = np.zeros(6)
            d[k] = 1e-6
            fd[k] = (oracle.inner_product(pr, X, Z, oracle.compose(oracle.exp(d), T), p) -
                     oracle.inner_product(pr, X, Z, oracle.compose(oracle.exp(-d), T), p)) / 2e-6
        assert np.linalg.norm(ev.grad - fd) <= 1e-4 * np.linalg.norm(fd)


# ------------------------------------------------------------ edge cases
def test_single_point_known_answers(ctx):
    one = PointCloud([[0.5, 0.5, 0.5]])
    p = KernelParams(lengthscale=0.1)
    pr = api.build_pairs(one, one, Isometry(), p, 3.0, 1e-4)
    off, idx, cf = pr.export()
    assert pr.size() == 1 and idx[0] == 0 and cf[0] == 1.0
    assert pr.cutoff_radius == pytest.approx(0.3)
    a, b = PointCloud([[0, 0, 0]]), PointCloud([[0.5, 0, 0]])
    p = KernelParams(lengthscale=0.5)
    assert api.indicator(a, a, Isometry(), p) == pytest.approx(1.0, rel=1e-6)
    assert api.indicator(a, b, Isometry(), p) == pytest.approx(0.6065306597126334, rel=1e-6)
    c = PointCloud([[1.5, 0, 0]])
    pr = api.build_pairs(a, c, Isometry(), p, 3.0, 0.0)
    assert api.inner_product(pr, a, c, Isometry(), p) == pytest.approx(0.011108996538242306, rel=1e-5)
    # lone point pulled toward the target, no torque (test_inner_product.cpp:174-189)
    z = PointCloud([[0.4, 0, 0]])
    pr = api.build_pairs(a, z, Isometry(), p, 10.0, 0.0)
    g = api.gradient(pr, a, z, Isometry(), p)
    assert g[3] < 0 and abs(g[4]) < 1e-12 and abs(g[5]) < 1e-12 and np.linalg.norm(g[:3]) < 1e-9


def test_empty_and_far_clouds(ctx):
    p = KernelParams(lengthscale=0.1)
    empty = PointCloud(np.zeros((0, 3)))
    pr = api.build_pairs(empty, empty, Isometry(), p, 3.0, 1e-4)
    assert pr.empty() and len(pr.export()[0]) == 1
    a, b = PointCloud([[0, 0, 0]]), PointCloud([[100, 0, 0]])
    assert api.build_pairs(a, b, Isometry(), p, 3.0, 1e-4).empty()
    with pytest.raises(ValueError):
        api.indicator(empty, a, Isometry(), p)
    cfg = RegistrationConfig(init_lengthscale=0.1, min_lengthscale=0.05, subsequent_lengthscale=0.1,
                             stabilization_window=3, max_iterations=600)
    with pytest.raises(NoOverlapError) as e:
        api.register_clouds(a, PointCloud([[1000, 0, 0]]), Isometry(), KernelParams(), cfg)
    assert e.value.cutoff_radius == pytest.approx(0.3) and "cutoff" in str(e.value)


def test_argument_errors(ctx):
    plain = PointCloud([[0, 0, 0]])
    colored = synth.random_labeled_cloud(3, 5, 1.0, True)
    p = KernelParams(lengthscale=0.1)
    with pytest.raises(ValueError, match="schema"):
        api.build_pairs(plain, colored, Isometry(), p, 3.0, 1e-4)
    with pytest.raises(ValueError):
        api.build_pairs(plain, plain, Isometry(), p, 0.5, 1e-4)
    with pytest.raises(ValueError):
        api.build_pairs(plain, plain, Isometry(), p, 3.0, 1.0)
    with pytest.raises(ValueError, match="decay_factor"):
        api.check_config(RegistrationConfig(decay_factor=1.5))
    with pytest.raises(ValueError, match="schema"):
        api.register_clouds(plain, colored, Isometry(), p, RegistrationConfig())


def test_orthogonal_semantics_dropped(ctx):
    sch = FeatureSchema([Channel("sem", 3, ChannelKind.semantic)])
    u = PointCloud([[0, 0, 0]], sch, [[1.0, 0, 0]])
    v = PointCloud([[0, 0, 0]], sch, [[0, 1.0, 0]])
    pl = KernelParams(lengthscale=0.5, per_channel=[ChannelParams(1.0, 1.0, KernelForm.linear)])
    assert api.build_pairs(u, v, Isometry(), pl, 3.0, 1e-9).size() == 0


def test_self_registration_is_identity(ctx):
    # test_registration.cpp:130-145 (tolerance-restated: FP32 device sums)
    C = synth.random_labeled_cloud(123, 150, 1.0, True)
    p = synth.params_for(C, 0.2, 0.3)
    cfg = RegistrationConfig(init_lengthscale=0.2, min_lengthscale=0.2, subsequent_lengthscale=0.2,
                             stabilization_window=3, max_iterations=600)
    res = api.register_clouds(C, C, Isometry(), p, cfg)
    assert res.converged
    assert rotation_angle(res.transform) <= 1e-4 and translation_norm(res.transform) <= 1e-4


def test_anneal_and_line_search_contract(ctx):
    cfg = RegistrationConfig(stabilization_window=5, stabilization_rel_tol=1e-5, min_lengthscale=0.01)
    assert api.anneal_step(0.5, [0.73] * 8, cfg) == 0.5 * 0.98
    assert api.anneal_step(0.0101, [0.73] * 8, cfg) == 0.0101
    X, Z = PointCloud([[0, 0, 0]]), PointCloud([[0.3, 0, 0]])
    p = KernelParams(lengthscale=0.5)
    pr = api.build_pairs(X, Z, Isometry(), p, 10.0, 0.0)
    g = api.gradient(pr, X, Z, Isometry(), p)
    eps = api.line_search(X, Z, Isometry(), g, p, pr, RegistrationConfig())
    assert eps > 0
    stepped = api.se3_compose(api.se3_exp(g * (eps / np.linalg.norm(g))), Isometry())
    assert api.inner_product(pr, X, Z, stepped, p) > api.inner_product(pr, X, Z, Isometry(), p)
    with pytest.raises(ValueError):
        api.line_search(X, Z, Isometry(), np.zeros(6), p, pr, RegistrationConfig())


def test_deterministic_and_batch_independent(ctx):
    X, Z, Ts = synth.kitti_pair(21, 8000)
    p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
    init = synth.perturbed(Ts, 2)
    a = api.register_clouds(X, Z, init, p, cfg)
    b = api.register_clouds(X, Z, init, p, cfg)
    assert np.array_equal(a.objective_trace, b.objective_trace) and np.array_equal(a.transform.as12(), b.transform.as12())
    X2, Z2, T2 = synth.kitti_pair(22, 8000)
    res, st = api.register_batch([X, X2], [Z, Z2], [init, synth.perturbed(T2, 3)], p, cfg)
    assert list(st) == [0, 0]
    assert np.array_equal(res[0].objective_trace, a.objective_trace)
    assert np.array_equal(res[0].transform.as12(), a.transform.as12())


def test_sweep_list_refilter_matches_candidate_filter(ctx):
    """Opt-in refilter (KREG_REFILTER=1): at annealing steps whose move since
    the last build is below the cutoff shrink, the new list is filtered from
    the resident sweep list. Same predicate on the same entries in the same
    order, so the registrations are bit-identical to the default path."""
    X, Z, Ts = synth.kitti_pair(7, 10000)  # converges in ~400 iterations, ~26 refilters
    p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
    init = synth.perturbed(Ts, 5)
    a = api.register_clouds(X, Z, init, p, cfg)
    os.environ["KREG_REFILTER"] = "1"
    try:
        c2 = api.Context()
    finally:
        del os.environ["KREG_REFILTER"]
    try:
        c2.reset_stats()
        b = api.register_clouds(X, Z, init, p, cfg, ctx=c2)
        assert c2.build_stats()["refilter_builds"] > 0
        assert np.array_equal(a.objective_trace, b.objective_trace)
        assert np.array_equal(a.pair_count_trace, b.pair_count_trace)
        assert np.array_equal(a.transform.as12(), b.transform.as12())
    finally:
        c2.close()


def test_host_buffer_batch_matches_device_batch(ctx):
    """register_batch_host (clouds staged on host threads, uploaded into the
    context arena) gives bitwise the results of register_batch."""
    Xs, Zs, inits = [], [], []
    for s in (31, 32, 33):
        X, Z, T = synth.kitti_pair(s, 6000)
        Xs.append(X)
        Zs.append(Z)
        inits.append(synth.perturbed(T, s))
    p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
    a, sa = api.register_batch(Xs, Zs, inits, p, cfg)
    for _ in range(2):  # the arena is reused by the second call
        b, sb = api.register_batch_host(Xs, Zs, inits, p, cfg)
        assert list(sa) == list(sb) == [0, 0, 0]
        for ra, rb in zip(a, b):
            assert np.array_equal(ra.transform.as12(), rb.transform.as12())
            assert np.array_equal(ra.objective_trace, rb.objective_trace)


def test_host_buffer_single_matches_device(ctx):
    """register_clouds_host (one pair staged into the context's upload arena,
    the CLI path) gives bitwise the result of register_clouds, call after call."""
    X, Z, T = synth.kitti_pair(41, 6000)
    init = synth.perturbed(T, 41)
    p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
    a = api.register_clouds(X, Z, init, p, cfg)
    for _ in range(2):
        b = api.register_clouds_host(X, Z, init, p, cfg)
        assert np.array_equal(a.transform.as12(), b.transform.as12())
        assert np.array_equal(a.objective_trace, b.objective_trace)


def test_kitti_registration_end_to_end_vs_reference(ctx, ref):
    X, Z, Ts = synth.kitti_pair(7, 40000)
    p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
    init = synth.perturbed(Ts, 3)
    ref.set_threads(max(1, os.cpu_count() or 1))
    r = ref.register_clouds(X, Z, init, p, cfg)
    ctx.reset_stats()
    g = api.register_clouds(X, Z, init, p, cfg)
    # the displacement screen answered most sweeps from its bound (no FP64
    # displacement pass) and the decisions below are still the reference's
    sc = ctx.screen_stats()
    assert sc["asked"] > 0 and sc["screened"] > sc["asked"] // 2, sc
    err = compose(inverse(g.transform), r.transform)
    assert rotation_angle(err) <= 1e-3 and translation_norm(err) <= 1e-3, (rotation_angle(err), translation_norm(err))
    assert g.converged == r.converged
    # decision-level parity on this pair: the same iterations, annealing
    # levels, accepted steps and rebuilds as the reference loop, F within 1e-6
    assert g.iterations == r.iterations
    assert np.array_equal(g.lengthscale_trace, r.lengthscale_trace)
    assert np.array_equal(g.step_trace, r.step_trace)
    assert np.array_equal(g.rebuild_trace, r.rebuild_trace)
    assert np.allclose(g.objective_trace, r.objective_trace, rtol=1e-6, atol=0)


def test_sequence_fallback_and_chains(ctx):
    base = synth.make_box_cloud(111, 150, False)
    empty = PointCloud(np.zeros((0, 3)))
    cfg = RegistrationConfig(init_lengthscale=0.15, min_lengthscale=0.15, subsequent_lengthscale=0.15,
                             stabilization_window=3, max_iterations=600)
    seq = api.register_sequence([base, base, empty, base], KernelParams(), cfg)
    assert list(seq.fallback) == [0, 1, 1] and len(seq.trajectory) == 4
    with pytest.raises(ValueError):
        api.register_sequence([base], KernelParams(), cfg)
    frames, poses = synth.kitti_sequence(5, 5, 6000)
    p, c2 = synth.kitti_params(), synth.kitti_subsequent_config()
    one = api.register_sequence(frames, p, c2)
    two = api.register_sequence(frames, p, c2, chains=2)
    assert len(two.relative) == 4 and not any(two.fallback)
    # chain 0 covers pairs (0,1),(1,2): identical to the single-chain run
    for k in range(2):
        assert np.array_equal(one.relative[k].as12(), two.relative[k].as12())

    # distributed chains (parallel.py): each "rank" runs its span block; the
    # assembled result equals the single-process chained run
    from paper_2012_03683_b200 import parallel
    spans = parallel.chain_spans(len(frames), 2)
    parts = []
    for r in range(2):
        mine = parallel.rank_spans(spans, r, 2)
        res = api.register_sequence_spans(frames, mine, p, c2)
        parts.append([(q, res.relative[q].as12().tolist(), int(res.fallback[q]), int(res.converged[q]),
                       float(res.final_indicator[q]), int(res.iterations[q])) for b, e in mine for q in range(b, e)])
        untouched = [q for q in range(len(frames) - 1) if not any(b <= q < e for b, e in mine)]
        assert all(np.array_equal(res.relative[q].as12(), Isometry().as12()) for q in untouched)
    merged = parallel.assemble_sequence(len(frames), parts)
    for k in range(len(frames) - 1):
        assert np.array_equal(merged.relative[k].as12(), two.relative[k].as12())
        assert np.allclose(merged.trajectory[k + 1].as12(), two.trajectory[k + 1].as12(), atol=1e-12)
    assert list(merged.iterations) == list(two.iterations)


def test_row_sharded_entry_point_single_rank(ctx):
    """kreg_register_clouds_rows with all rows and no collective is
    register_clouds (C4 row sharding degenerates to one rank)."""
    X, Z, Ts = synth.kitti_pair(23, 6000)
    p, cfg = synth.kitti_params(), synth.kitti_subsequent_config()
    init = synth.perturbed(Ts, 4)
    a = api.register_clouds(X, Z, init, p, cfg)
    b = api.register_clouds_rows(X, Z, Z.size(), init, p, cfg)
    assert np.array_equal(a.transform.as12(), b.transform.as12())
    assert np.array_equal(a.objective_trace, b.objective_trace)
    # a half-row share with the full denominator: indicator uses sqrt(|X| |Z|)
    from paper_2012_03683_b200 import parallel
    half = parallel.shard_rows(Z, 0, 2)
    c = api.register_clouds_rows(X, half, Z.size(), init, p, cfg)
    assert c.indicator_trace[0] == pytest.approx(c.objective_trace[0] / math.sqrt(X.size() * Z.size()), rel=1e-12)
    with pytest.raises(ValueError):
        api.register_clouds_rows(X, Z, Z.size() - 1, init, p, cfg)


# -------------------------------------------- K4 dense exact cosine
def test_exact_cosine_reference_cases(ctx, ref):
    # test_inner_product.cpp:314-350 on the device
    C_ = synth.random_labeled_cloud(71, 60, 1.0, True, 3)
    p = synth.params_for(C_, 0.3, 0.3)
    assert api.exact_cosine(C_, C_, Isometry(), p) == pytest.approx(1.0, abs=1e-14)
    a, b = PointCloud([[0.0, 0.0, 0.0]]), PointCloud([[0.5, 0.0, 0.0]])
    assert api.exact_cosine(a, b, Isometry(), KernelParams(lengthscale=0.5)) == pytest.approx(0.6065306597126334,
                                                                                            rel=1e-12)
    X = synth.random_labeled_cloud(81, 100, 1.0, True, 3)
    Z = synth.random_labeled_cloud(82, 100, 1.0, True, 3)
    T = synth.random_isometry(synth.SplitMix64(83), 0.3, 0.2)
    p = synth.params_for(X, 0.25, 0.3)
    assert api.exact_cosine(X, Z, T, p) == pytest.approx(ref.exact_cosine(X, Z, T, p), rel=1e-12)
    schema = FeatureSchema([Channel("sem", 2, ChannelKind.semantic)])
    zero = PointCloud([[0.0, 0.0, 0.0]], schema, np.zeros((1, 2)))
    with pytest.raises(ValueError):
        api.exact_cosine(zero, zero, Isometry(), KernelParams(lengthscale=0.5,
                                                              per_channel=[ChannelParams(1.0, 1.0, KernelForm.linear)]))
    with pytest.raises(ValueError):
        api.exact_cosine(PointCloud(np.zeros((0, 3))), a, Isometry(), KernelParams())


def test_exact_cosine_kitti_vs_reference(ctx, ref):
    X, Z, Ts = synth.kitti_pair(9, 3000)
    p = synth.kitti_params()
    for T in (Ts, synth.perturbed(Ts, 2, 0.05, 0.2)):
        got, parts = api.exact_cosine(X, Z, T, p, parts=True)
        want = ref.exact_cosine(X, Z, T, p)
        assert got == pytest.approx(want, rel=1e-12)
        assert 0.0 < got < 1.0 and all(v > 0 for v in parts)


def test_indicator_sweep_vs_reference(ctx, ref):
    """eval.cpp:198-235 indicator_sweep: indicator(cloud, P cloud, I) at evenly
    spaced magnitudes == the reference's indicator(cloud, cloud, P)."""
    X, _, _ = synth.kitti_pair(13, 4000)
    p = synth.kitti_params()
    cen = X.positions.mean(axis=0)
    for axis, rng_ in (("rotation", 0.05), ("translation", 0.2)):
        rows = api.indicator_sweep(X, p, axis, rng_, 5)
        assert [m for m, _ in rows] == pytest.approx([rng_ * k / 4 for k in range(5)], abs=1e-15)
        for m, ind in rows:
            if axis == "rotation":
                R = api.se3_exp([0, 0, m, 0, 0, 0])
                P = Isometry(R.rotation, cen - R.rotation @ cen)
            else:
                P = Isometry(np.eye(3), np.array([m, 0.0, 0.0]))
            want = ref.indicator(X, X, P, p)
            assert ind == pytest.approx(want, rel=1e-4)
        inds = [v for _, v in rows]
        assert inds[0] > inds[-1]  # misalignment lowers the indicator
    assert len(api.indicator_sweep(X, p, "translation", 0.0, 1)) == 1
    with pytest.raises(ValueError):
        api.indicator_sweep(X, p, "rotation", 0.1, 1)
    with pytest.raises(ValueError):
        api.indicator_sweep(X, p, "rotation", -0.1, 3)


def test_tum_registration_vs_reference(ctx, ref):
    """C2 (TUM-shaped 20k, colour dim 5) registration: same decisions as the
    reference loop (iterations, levels) and the same pose to 1e-3."""
    X, Z, Ts = synth.tum_pair(5, 20000)
    p, cfg = synth.tum_params(), synth.tum_subsequent_config()
    ref.set_threads(max(1, os.cpu_count() or 1))
    r = ref.register_clouds(X, Z, Isometry(), p, cfg)
    g = api.register_clouds(X, Z, Isometry(), p, cfg)
    err = compose(inverse(g.transform), r.transform)
    assert rotation_angle(err) <= 1e-3 and translation_norm(err) <= 1e-3, (rotation_angle(err), translation_norm(err))
    assert g.converged == r.converged
    assert abs(g.iterations - r.iterations) <= max(2, r.iterations // 50)
    assert np.allclose(g.objective_trace[:20], r.objective_trace[:20], rtol=1e-6, atol=0)
