"""Development probe: per-warp event timeline (clock64) of CTA 0 of the factor kernel over the
sweep steps of line 10 (profiling build, FFB_PROFILE=1)."""
import ctypes as C
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_02977_b200 import flowfem as ff, synth, _lib  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
f0, f1, _, cfg = synth.make(name)
lib = _lib.load()
lib.ffb_debug_prof.argtypes = [C.c_void_p, C.c_int]
ctx = ff.Context(0)
rc = ff.RunConfig(sigma=cfg.sigma, parts=cfg.parts, overlap=cfg.overlap, adapt_iters=0, cg_tolerance=cfg.tol)
r = ff.run_on_frames(f0, f1, rc, ctx)
buf = (C.c_ulonglong * (16 * 16 * 8))()
lib.ffb_debug_prof(buf, 3)
a = np.frombuffer(buf, dtype=np.uint64).reshape(16, 16, 8).astype(np.int64)
# warps >= 4: "kk" = Z loop done before the barrier, "pivot" = first Z row block stored
names = ["start", "Zdone", "kk", "pivot", "tiles", "end"]
print(f"{name}: factor {r.stats.ms_factor:.1f} ms")
for st in range(2, 5):
    base = a[st, 0, 0]
    print(f"step {st}: next step start at {a[st + 1, 0, 0] - base}")
    for w in range(16):
        row = [a[st, w, i] - base if a[st, w, i] else None for i in range(6)]
        ark, rup = a[st, w, 6], a[st, w, 7]
        extra = f" | ark {ark // 16:6d} cyc/{ark % 16} tiles, rupd {rup // 16:6d} cyc/{rup % 16} tiles"
        print(f"  w{w:2d} " + " ".join(f"{n}={v:7d}" if v is not None and abs(v) < 10**8 else f"{n}=    -  " for n, v in zip(names, row)) + extra)
print("step period:", np.diff(a[:10, 0, 0]).tolist())
