"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference.

The reference is compiled from /root/reference/proj/src by oracle/Makefile
(target `ref`) into oracle/_ref/libkreg_ref.so; this script calls it through
oracle/ref/ref_capi.cpp and stores inputs + outputs as small .npz files, so
the parity tests can run on a machine without the reference tree.

    make -C oracle ref && python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from _checkers import Reference  # noqa: E402
from paper_2012_03683_b200 import synth  # noqa: E402
from paper_2012_03683_b200.types import Isometry, RegistrationConfig  # noqa: E402


def cloud_arrays(prefix, c):
    return {f"{prefix}_xyz": c.positions, f"{prefix}_feat": c.features}


def params_arrays(p):
    return {"sigma": p.sigma, "lengthscale": p.lengthscale,
            "per_channel": np.array([[cp.sigma, cp.lengthscale, int(cp.form)] for cp in p.per_channel]).reshape(-1, 3)}


def main():
    r = Reference()
    r.set_threads(4)
    meta = {}

    # 1. grid search == brute force (test_inner_product.cpp:90-105), F/grad
    for seed in (101, 102, 103):
        X = synth.random_labeled_cloud(seed, 500, 1.0, True)
        Z = synth.random_labeled_cloud(seed + 50, 500, 1.0, True)
        rng = synth.SplitMix64(seed)
        T = synth.random_isometry(rng, 0.3, 0.2)
        p = synth.params_for(X, 0.08, 0.3)
        pr = r.build_pairs(X, Z, T, p, 3.0, 1e-4)
        ev = r.objective_and_gradient(pr, X, Z, T, p)
        np.savez_compressed(os.path.join(HERE, f"labeled_{seed}.npz"), **cloud_arrays("X", X), **cloud_arrays("Z", Z),
                            T=T.as12(), offsets=pr.offsets, x_index=pr.x_index, coeff=pr.coeff, eval=ev,
                            **params_arrays(p))

    # 2. KITTI-shaped small pair: pair sets + F/grad at several T and l, and a
    #    full registration with the subsequent-frame KITTI schedule
    X, Z, Ts = synth.kitti_pair(11, 3000)
    init = synth.perturbed(Ts, 5)
    p = synth.kitti_params()
    cfg = synth.kitti_subsequent_config()
    Tlist = [init, Ts, synth.perturbed(Ts, 9, math.radians(1.0), 0.1)]
    evals, counts = [], []
    for l in (0.1, 0.0475):
        pl = p.with_lengthscale(l)
        for T in Tlist:
            pr = r.build_pairs(X, Z, T, pl, 3.0, 1e-4)
            counts.append(pr.size())
            evals.append(r.objective_and_gradient(pr, X, Z, T, pl))
    pr = r.build_pairs(X, Z, init, p.with_lengthscale(0.1), 3.0, 1e-4)
    res = r.register_clouds(X, Z, init, p, cfg)
    np.savez_compressed(os.path.join(HERE, "kitti_small.npz"), **cloud_arrays("X", X), **cloud_arrays("Z", Z),
                        T_star=Ts.as12(), init=init.as12(), Tlist=np.stack([T.as12() for T in Tlist]),
                        evals=np.array(evals), counts=np.array(counts),
                        offsets=pr.offsets, x_index=pr.x_index, coeff=pr.coeff,
                        reg_T=res.transform.as12(), reg_iterations=res.iterations, reg_converged=res.converged,
                        reg_objective=res.objective_trace, reg_lengthscale=res.lengthscale_trace,
                        reg_pairs=res.pair_count_trace, reg_final_indicator=res.final_indicator)
    meta["kitti_small"] = {"iterations": res.iterations, "converged": res.converged}

    # 3. box recovery (test_registration.cpp:147-170 shape), geometric-only
    Xb = synth.make_box_cloud(2024, 500, False)
    rng = synth.SplitMix64(11)
    axis = synth._normalized([rng.gaussian(), rng.gaussian(), rng.gaussian()])
    Tst = synth.se3_exp(np.concatenate([axis * (5.0 * math.pi / 180.0), [0, 0, 0]]))
    diam = r.diameter(Xb)
    Tst = Isometry(Tst.rotation, 0.05 * diam * np.array(synth._normalized([rng.gaussian(), rng.gaussian(), rng.gaussian()])))
    from paper_2012_03683_b200.types import inverse, PointCloud, KernelParams
    Zb = PointCloud(inverse(Tst).apply(Xb.positions))
    cfgb = RegistrationConfig(init_lengthscale=0.12, min_lengthscale=0.08, subsequent_lengthscale=0.12,
                              stabilization_window=3, max_iterations=600)
    resb = r.register_clouds(Xb, Zb, Isometry(), KernelParams(), cfgb)
    np.savez_compressed(os.path.join(HERE, "box_registration.npz"), X_xyz=Xb.positions, Z_xyz=Zb.positions,
                        T_star=Tst.as12(), reg_T=resb.transform.as12(), reg_iterations=resb.iterations,
                        reg_converged=resb.converged, reg_objective=resb.objective_trace,
                        reg_lengthscale=resb.lengthscale_trace, reg_step=resb.step_trace)
    meta["box"] = {"iterations": resb.iterations, "converged": resb.converged}

    # 4. known answers quoted by the reference tests
    meta["known_answers"] = {
        "k_one_lengthscale": 0.6065306597126334,   # test_kernels.cpp:14-16
        "k_three_lengthscales": 0.011108996538242306,  # test_kernels.cpp:18-20
    }
    with open(os.path.join(HERE, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
