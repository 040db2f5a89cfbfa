"""Positive control of the bounds-check variant (KREG_DEBUG_BOUNDS + KREG_BOUNDS_SELFTEST):
a deliberately failing check must be counted (site 99)."""
import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
from paper_2012_03683_b200 import api, synth
X, Z, Ts = synth.kitti_pair(7, 5000)
api.build_pairs(X, Z, Ts, synth.kitti_params(), 3.0, 1e-4)
lib = api.lib()
lib.kreg_debug_violations.restype = C.c_longlong
lib.kreg_debug_violations.argtypes = [C.POINTER(C.c_int)]
s = C.c_int(0)
print("selftest violations", lib.kreg_debug_violations(C.byref(s)), "site", s.value)
