"""Development probe: per-phase clock64 accounting of the factor/solve kernels for one
configuration (library built with FFB_PROFILE=1)."""
import ctypes as C
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_02977_b200 import flowfem as ff, synth, _lib
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
f0, f1, _, cfg = synth.make(name)
lib = _lib.load()
lib.ffb_debug_prof.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 64)()
ctx = ff.Context(0)
rc = ff.RunConfig(sigma=cfg.sigma, parts=cfg.parts, overlap=cfg.overlap, adapt_iters=0, cg_tolerance=cfg.tol)
ff.run_on_frames(f0, f1, rc, ctx)
lib.ffb_debug_prof(buf, 1)
r = ff.run_on_frames(f0, f1, rc, ctx)
lib.ffb_debug_prof(buf, 1)
print(name, "factor ms", r.stats.ms_factor, "pcg ms", r.stats.ms_pcg, "iters", r.stats.iters)
fn = ["buildD", "pivot", "Z", "Rupd", "X+sync", "line"]
vals = [buf[0], buf[33], buf[34], buf[35], buf[36], buf[5]]
tot = sum(vals) or 1
print("factor CTA0 cycles:", {fn[i]: f"{vals[i]/1e6:.1f}M ({100*vals[i]/tot:.0f}%)" for i in range(6)})
print("  warp0: kk tile %.1fM pivot %.1fM (top sync %.1fM) X-work %.1fM" % (buf[38]/1e6, buf[37]/1e6, buf[33]/1e6, buf[39]/1e6))
sn = ["operand", "fullwait", "rows", "colflush", "reduce+sync", "owner+sync"]
tot = sum(buf[16 + i] for i in range(6)) or 1
print("solve CTA0 cycles:", {sn[i]: f"{buf[16+i]/1e6:.2f}M ({100*buf[16+i]/tot:.0f}%)" for i in range(6)})
