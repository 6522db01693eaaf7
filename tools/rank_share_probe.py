"""Development probe: the subdomain-solve application time of ONE rank's share of c4 at 8 GPUs
(32 subdomains = 2 subdomain rows of the 16x16 partition: a 270x3840 frame pair cut 16x2, same
subdomain size), for the solve cluster sizes given on the command line (FFB_CLUSTER is read when
the partition is set, so each size runs in its own context)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_02977_b200 import flowfem as ff, synth, _lib  # noqa: E402

H, W, parts = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (270, 3840, 32)
f0, f1, _ = synth.gen_c3(0, H, W)
lib = _lib.load()
lib.ffb_debug_time_asm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
for cl in (sys.argv[4:] or ["1", "2"]):
    os.environ["FFB_CLUSTER"] = cl
    ctx = ff.Context(0)
    rc = ff.RunConfig(sigma=1.5, parts=parts, overlap=4, adapt_iters=0, cg_tolerance=1e-10)
    r = ff.run_on_frames(f0, f1, rc, ctx)
    gb = 8 * r.stats.factor_doubles / 1e9
    ms = C.c_double()
    assert lib.ffb_debug_time_asm(ctx.handle, 3, 100, 0, C.byref(ms)) == 0, _lib.last_error()
    print(f"{H}x{W} parts {r.stats.parts_x}x{r.stats.parts_y} cluster {cl}: {ms.value:.3f} ms/application, "
          f"{1e3 * gb / ms.value:.0f} GB/s; factor {r.stats.ms_factor:.1f} ms, iters {r.stats.iters}", flush=True)
    del ctx
