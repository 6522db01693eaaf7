"""Development probe: time the Schwarz preconditioner application alone for a configuration
(after one full solve), optionally under FFB_SOLVE_DBG decomposition flags."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_02977_b200 import flowfem as ff, synth, _lib  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
f0, f1, _, cfg = synth.make(name)
lib = _lib.load()
lib.ffb_debug_time_asm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
ctx = ff.Context(0)
rc = ff.RunConfig(sigma=cfg.sigma, parts=cfg.parts, overlap=cfg.overlap, adapt_iters=0,
                  cg_tolerance=cfg.tol)
r = ff.run_on_frames(f0, f1, rc, ctx)
gb = 8 * r.stats.factor_doubles / 1e9
for dbg in [int(a) for a in (sys.argv[2:] or ["0"])]:
    ms = C.c_double()
    assert lib.ffb_debug_time_asm(ctx.handle, 3, 50, dbg, C.byref(ms)) == 0, _lib.last_error()
    print(f"{name} dbg={dbg} C={os.environ.get('FFB_CLUSTER', 'auto')}: "
          f"{ms.value:.3f} ms/application, {1e3 * gb / ms.value:.0f} GB/s")
