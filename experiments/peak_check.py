import sys, ctypes
sys.path.insert(0, '/root/repo')
from paper_2604_11599_b200 import _lib
ctx = _lib.context()
for i in range(5):
    v = ctypes.c_double()
    _lib.check(ctx.lib.qsb_debug_fma_peak(ctx.handle, _lib.C128, ctypes.byref(v)))
    print("fp64", v.value)
