"""Bounds-check run (diagnostic): the GPU test suite plus a large pair through
the KREG_DEBUG_BOUNDS variant, then the device violation counter must be 0.

    python -c "from paper_2012_03683_b200.build import build_variant as b; b('bounds', ['KREG_DEBUG_BOUNDS'])"
    KREG_LIB=paper_2012_03683_b200/_variants/bounds.so python tools/bounds_check.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.getcwd())
import pytest  # noqa: E402

from paper_2012_03683_b200 import api, synth  # noqa: E402

assert "bounds" in os.environ.get("KREG_LIB", ""), "run with KREG_LIB=<bounds variant>"
rc = pytest.main(["-q", "-m", "gpu", "-x", "tests"])
lib = api.lib()
lib.kreg_debug_violations.restype = C.c_longlong
lib.kreg_debug_violations.argtypes = [C.POINTER(C.c_int)]
site = C.c_int(0)
n_tests = lib.kreg_debug_violations(C.byref(site))
print("violations after the GPU suite:", n_tests, "site", site.value, flush=True)
# a large pair: many chunks per list, big candidate rows
X, Z, Ts = synth.kitti_pair(2012, 400000)
res = api.register_clouds(X, Z, synth.perturbed(Ts, 4), synth.kitti_params(), synth.kitti_subsequent_config())
n_big = lib.kreg_debug_violations(C.byref(site))
print("violations on a 400k-point registration:", n_big, "site", site.value, "iterations", res.iterations, flush=True)
sys.exit(0 if rc == 0 and n_tests == 0 and n_big == 0 else 1)
