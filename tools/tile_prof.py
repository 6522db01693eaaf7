"""Development probe: per-phase clock64 accounting of the register-tiled solve kernel (CTA 0,
warp 0 = tile (0,0) + owner of block 0), profiling build (FFB_PROFILE=1)."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_02977_b200 import flowfem as ff, synth, _lib  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
f0, f1, _, cfg = synth.make(name)
lib = _lib.load()
lib.ffb_debug_prof.argtypes = [C.c_void_p, C.c_int]
lib.ffb_debug_time_asm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
buf = (C.c_ulonglong * 64)()
ctx = ff.Context(0)
rc = ff.RunConfig(sigma=cfg.sigma, parts=cfg.parts, overlap=cfg.overlap, adapt_iters=0, cg_tolerance=cfg.tol)
ff.run_on_frames(f0, f1, rc, ctx)
lib.ffb_debug_prof(buf, 1)
ms = C.c_double()
n = 50
assert lib.ffb_debug_time_asm(ctx.handle, 3, n, 0, C.byref(ms)) == 0
lib.ffb_debug_prof(buf, 1)
names = ["xwait", "operand+bar", "fma", "shfl", "load+send", "blkwait", "sum+bcast"]
tot = sum(buf[48 + i] for i in range(7)) or 1
print(f"{name}: {ms.value:.3f} ms/application")
print({names[i]: f"{buf[48+i]/1e6:.2f}M ({100*buf[48+i]/tot:.0f}%)" for i in range(7)})
