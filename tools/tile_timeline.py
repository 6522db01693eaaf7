"""Development probe: per-warp event timeline (clock64) of CTA 0 of the register-tiled solve
kernel over forward line steps 8..23 (profiling build, FFB_PROFILE=1)."""
import ctypes as C
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_02977_b200 import flowfem as ff, synth, _lib  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
dbg = int(sys.argv[2]) if len(sys.argv) > 2 else 0
f0, f1, _, cfg = synth.make(name)
lib = _lib.load()
lib.ffb_debug_prof.argtypes = [C.c_void_p, C.c_int]
lib.ffb_debug_time_asm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
ctx = ff.Context(0)
rc = ff.RunConfig(sigma=cfg.sigma, parts=cfg.parts, overlap=cfg.overlap, adapt_iters=0, cg_tolerance=cfg.tol)
ff.run_on_frames(f0, f1, rc, ctx)
ms = C.c_double()
assert lib.ffb_debug_time_asm(ctx.handle, 3, 3, dbg, C.byref(ms)) == 0
buf = (C.c_ulonglong * (16 * 16 * 8))()
lib.ffb_debug_prof(buf, 2)
a = np.frombuffer(buf, dtype=np.uint64).reshape(16, 16, 8).astype(np.int64)
names = ["x_ok", "bar", "fma", "shfl", "sent", "own_in", "own_out", "data"]
print(f"{name} dbg={dbg}: {ms.value:.3f} ms/application")
for t in range(4, 8):
    base = a[t, 0, 0]
    print(f"line {t + 8}: (cycles after warp 0 x_ok; next line x_ok at {a[t + 1, 0, 0] - base})")
    for w in range(16):
        row = [a[t, w, i] - base if a[t, w, i] else None for i in range(8)]
        print(f"  w{w:2d} " + " ".join(f"{n}={v:6d}" if v is not None and abs(v) < 10**7 else f"{n}=   -  " for n, v in zip(names, row)))
per = np.diff(a[:, 0, 0])
print("line period (cycles):", per[:15].tolist())
