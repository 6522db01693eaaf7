import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1508_02977_b200 import flowfem as ff, parallel as par
from paper_1508_02977_b200.synth import gen_c1
f0, f1, _ = gen_c1(0, 72, 96)
cfg = ff.RunConfig(sigma=1.0, parts=4, overlap=3, adapt_iters=0, cg_tolerance=1e-11)
st = torch.cuda.current_stream().cuda_stream
def mk(r, w):
    c = ff.Context(0); c.set_stream(st)
    b = par.DeviceBackend(c, r, w); b.setup(f0, f1, cfg); b.begin(3, 1e-11, 0, False); return b
single = mk(0, 1); pair = [mk(0, 2), mk(1, 2)]
zs = [b.z_buffer() for b in pair]
def red():
    tot = zs[0] + zs[1]; zs[0].copy_(tot); zs[1].copy_(tot)
def cmp(tag):
    torch.cuda.synchronize()
    for w, nm in ((0,'z'),(1,'r'),(2,'x'),(3,'p0'),(4,'p1')):
        a = single.z_buffer(w); d0 = float((a - pair[0].z_buffer(w)).abs().max()); d1 = float((a - pair[1].z_buffer(w)).abs().max())
        print(tag, nm, '%.2e %.2e' % (d0, d1), end=' | ')
    print()
red(); [b.stage(1) for b in pair]; single.stage(1); cmp('after-init')
single.stage(0)
for b in pair: b.stage(0)
cmp('stage0-before-reduce')
red(); cmp('after-reduce')
for b in pair: b.stage(1)
single.stage(1)
cmp('it0-stage1')
for it in range(1, 3):
    single.stage(0)
    for b in pair: b.stage(0)
    cmp(f'it{it}-stage0')
    red(); cmp(f'it{it}-reduce')
    single.stage(1)
    for b in pair: b.stage(1)
    cmp(f'it{it}-stage1')
