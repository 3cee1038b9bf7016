"""CTA-0 timeline of the sweep kernel (GABP_TIMELINE build):
GABP_LIB=.../libgabp_b200_tl.so python tools/timeline.py --config 2"""
import argparse, ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0810_1119_b200 as G
from paper_0810_1119_b200 import _lib, problems
ap = argparse.ArgumentParser(); ap.add_argument("--config", type=int, default=2)
ap.add_argument("--tiles", type=int, default=8); args = ap.parse_args()
lib = _lib.load()
lib.gabp_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
name, fn = problems.CONFIGS[args.config]
g = G.build_graph(fn(0).system, 0)
ms = ctypes.c_double()
_lib.check(lib.gabp_bench_sweeps(g.handle, 2, 4, ctypes.byref(ms)))
N = 64 * 9 * 8
tl = (ctypes.c_longlong * N)()
_lib.check(lib.gabp_debug_timeline(tl, N))
print(f"{name}: {ms.value:.3f} ms/sweep (timeline build)")
cons = ["loop", "full_ok", "gath_iss", "cp_wait", "bar_pre", "row_done", "comp_done", "bar_post"]
prod = ["loop", "empty_ok", "issued"]
base = min(v for v in tl if v > 0)
for k in range(2, 2 + args.tiles):
    for w in range(9):
        row = [tl[(k * 9 + w) * 8 + e] for e in range(8)]
        if row[0] == 0:
            continue
        names = prod if w == 4 else cons
        n = 3 if w == 4 else 8
        print(f"k={k:2d} w{w}: t0={row[0] - base:8d} " +
              " ".join(f"{names[e]}=+{row[e] - row[0]}" for e in range(1, n) if row[e]))
