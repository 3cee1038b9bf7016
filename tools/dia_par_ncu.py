import sys, ctypes; sys.path.insert(0,'.')
import paper_0810_1119_b200 as G
from paper_0810_1119_b200 import _lib, grid as GR
lib=_lib.load()
g = GR.GridGraph(GR.GridSpec(2, 4096, 0), 0)
ms=ctypes.c_double()
_lib.check(lib.gabp_bench_sweeps(g.handle, 0, 0, 8, ctypes.byref(ms)))
print(ms.value)
