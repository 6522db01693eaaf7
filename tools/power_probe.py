"""Development probe: power draw, SM clock and achieved bandwidth of (a) the Schwarz
preconditioner application alone in a sustained loop, (b) a plain device copy, (c) a read-only
reduction, each for several seconds — is the sustained solve power-capped below what a plain
stream sustains?"""
import ctypes as C
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_1508_02977_b200 import flowfem as ff, synth, _lib  # noqa: E402


class Sampler:
    def __init__(self):
        self.rows, self._stop = [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            out = subprocess.run(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.mem,power.draw",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout
            try:
                self.rows.append([float(v) for v in out.strip().split(",")])
            except ValueError:
                pass
            time.sleep(0.1)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join()

    def summary(self):
        r = self.rows[len(self.rows) // 3:] or [[0, 0, 0]]
        med = lambda k: sorted(x[k] for x in r)[len(r) // 2]
        return f"sm {med(0):.0f} MHz, mem {med(1):.0f} MHz, power {med(2):.0f} W ({len(r)} samples)"


name = sys.argv[1] if len(sys.argv) > 1 else "c4"
napp = int(sys.argv[2]) if len(sys.argv) > 2 else 300
f0, f1, _, cfg = synth.make(name)
lib = _lib.load()
lib.ffb_debug_time_asm.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
ctx = ff.Context(0)
rc = ff.RunConfig(sigma=cfg.sigma, parts=cfg.parts, overlap=cfg.overlap, adapt_iters=0, cg_tolerance=cfg.tol)
r = ff.run_on_frames(f0, f1, rc, ctx)
gb = 8 * r.stats.factor_doubles / 1e9
ms = C.c_double()
for n in (20, napp):
    with Sampler() as s:
        assert lib.ffb_debug_time_asm(ctx.handle, 3, n, 0, C.byref(ms)) == 0, _lib.last_error()
    print(f"{name} solve x{n}: {ms.value:.3f} ms/application, {1e3 * gb / ms.value:.0f} GB/s (factor bytes/s, fwd+bwd ~2x{gb:.1f} GB)  {s.summary()}", flush=True)

a = torch.empty(1 << 30, dtype=torch.float64, device="cuda")  # 8 GB
b = torch.empty_like(a)
a.fill_(1.0)
for label, fn, bytes_ in (("copy", lambda: b.copy_(a), 16 * (1 << 30)), ("sum (read-only)", lambda: a.sum(), 8 * (1 << 30))):
    for secs in (0.3, 6.0):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        with Sampler() as s:
            t0 = time.time(); k = 0
            e0.record()
            while time.time() - t0 < secs:
                for _ in range(10):
                    fn()
                k += 10
                torch.cuda.synchronize()
            e1.record(); torch.cuda.synchronize()
        print(f"{label} for {secs} s: {bytes_ * k / e0.elapsed_time(e1) / 1e6:.0f} GB/s  {s.summary()}", flush=True)
