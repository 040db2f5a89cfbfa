import os, sys
sys.path.insert(0, os.getcwd())
from paper_2012_03683_b200 import api, synth
X, Z, Ts = synth.kitti_pair(7, 40000)
pl = synth.kitti_params().with_lengthscale(0.1)
pr = api.build_pairs(X, Z, Ts, pl, 3.0, 1e-4)
for _ in range(5):
    api.eval_transforms(pr, X, Z, [Ts, Ts], pl)
print(pr.info())
