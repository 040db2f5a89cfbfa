import sys, time, os, math
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from paper_2012_03683_b200 import api, synth
from paper_2012_03683_b200.types import *
from _checkers import Oracle, Reference
o = Oracle(); r = Reference()
ctx = api.default_context()
z = np.load("tests/golden/box_registration.npz")
X, Z = PointCloud(z["X_xyz"]), PointCloud(z["Z_xyz"])
cfg = RegistrationConfig(init_lengthscale=0.12, min_lengthscale=0.08, subsequent_lengthscale=0.12, stabilization_window=3, max_iterations=600)
g = api.register_clouds(X, Z, Isometry(), KernelParams(), cfg)
rr = r.register_clouds(X, Z, Isometry(), KernelParams(), cfg)
print("iters gpu/ref", g.iterations, rr.iterations, g.converged, rr.converged)
n = min(g.iterations, rr.iterations)
rel = np.abs(g.objective_trace[:n] - rr.objective_trace[:n]) / rr.objective_trace[:n]
print("first obj rel diffs", rel[:10])
print("ls equal prefix", np.argmax(g.lengthscale_trace[:n] != rr.lengthscale_trace[:n]))
print("step gpu", g.step_trace[:12]); print("step ref", rr.step_trace[:12])
print("tail gpu", g.objective_trace[-5:], g.step_trace[-5:], g.twist_norm_trace[-5:])
print("tail ref", rr.objective_trace[-5:], rr.step_trace[-5:], rr.twist_norm_trace[-5:])
# F accuracy at final level
l = float(rr.lengthscale_trace[-1]); p = KernelParams(lengthscale=l)
Tr = rr.transform
pg = api.build_pairs(X, Z, Tr, p, 3.0, 1e-4); po = o.build_pairs(X, Z, Tr, p, 3.0, 1e-4)
print("pairs", pg.size(), po.size())
rng = synth.SplitMix64(3)
errs = []
for k in range(10):
    T = compose(synth.random_isometry(rng, 1e-3, 1e-3), Tr)
    a = api.eval_transforms(pg, X, Z, [T], p)[0]; b = o.objective_and_gradient(po, X, Z, T, p)
    errs.append(((a[0]-b[0])/b[0], np.linalg.norm(a[1:7]-b[1:])/np.linalg.norm(b[1:]), np.linalg.norm(b[1:])))
print("F rel err / g rel err / |g|", np.array(errs))
# line through the optimum along rotation about z
ts = np.linspace(-2e-3, 2e-3, 41)
Ts = [compose(synth.se3_exp([0, 0, t, 0, 0, 0]), Tr) for t in ts]
Fg = np.concatenate([api.eval_transforms(pg, X, Z, Ts[i:i+8], p)[:, 0] for i in range(0, 41, 8)])
Fo = np.array([o.inner_product(po, X, Z, T, p) for T in Ts])
print("Fo - Fo[20]", (Fo - Fo[20])[::5]); print("Fg - Fg[20]", (Fg - Fg[20])[::5]); print("Fg-Fo rel", ((Fg-Fo)/Fo)[::5])
Tg = g.transform
print("F_ref(Tref), F_ref(Tgpu)", o.inner_product(po, X, Z, Tr, p), o.inner_product(po, X, Z, Tg, p))
# perf: eval latency per call vs P
Xk, Zk, Ts_ = synth.kitti_pair(7, 40000); pk = synth.kitti_params()
for l in (0.1, 0.0475):
    pr = api.build_pairs(Xk, Zk, Ts_, pk.with_lengthscale(l), 3.0, 1e-4)
    for M in (1, 2, 4, 8):
        Tl = [Ts_] * M
        api.eval_transforms(pr, Xk, Zk, Tl, pk.with_lengthscale(l))
        t = time.perf_counter(); N = 50
        for _ in range(N): api.eval_transforms(pr, Xk, Zk, Tl, pk.with_lengthscale(l))
        dt = (time.perf_counter() - t) / N
        print(f"l={l} P={pr.size()} M={M} eval call {dt*1e6:.1f} us -> {pr.size()*M/dt/1e9:.1f} G pair-evals/s", flush=True)
    t = time.perf_counter()
    for _ in range(20): api.build_pairs(Xk, Zk, Ts_, pk.with_lengthscale(l), 3.0, 1e-4)
    print("build call", (time.perf_counter() - t) / 20 * 1e6, "us")
ctx.set_profiling(True); ctx.reset_stats()
pr = api.build_pairs(Xk, Zk, Ts_, pk.with_lengthscale(0.1), 3.0, 1e-4)
for _ in range(20): api.eval_transforms(pr, Xk, Zk, [Ts_] * 2, pk.with_lengthscale(0.1))
print(ctx.sweep_stats())
