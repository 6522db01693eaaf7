import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1508_02977_b200 import flowfem as ff, parallel as par
from paper_1508_02977_b200.synth import gen_c1
f0, f1, _ = gen_c1(0, 72, 96)
cfg = ff.RunConfig(sigma=1.0, parts=4, overlap=3, adapt_iters=0, cg_tolerance=1e-11)
st = torch.cuda.current_stream().cuda_stream
bs = []
for r, w in ((0, 1), (0, 2), (1, 2)):
    c = ff.Context(0); c.set_stream(st)
    b = par.DeviceBackend(c, r, w); b.setup(f0, f1, cfg); b.begin(3, 1e-11, 0, False)
    bs.append(b)
torch.cuda.synchronize()
z = [b.z_buffer().cpu().numpy() for b in bs]
print("full", np.abs(z[0]).max(), "r0", np.abs(z[1]).max(), "r1", np.abs(z[2]).max())
print("diff", np.abs(z[1] + z[2] - z[0]).max())
d = (z[1] + z[2] - z[0]).reshape(72, 96, 3)
print("bad pixels", np.argwhere(np.abs(d).max(axis=2) > 1e-12)[:10], (np.abs(d).max(axis=2) > 1e-12).sum())
t = bs[1].z_buffer()
t.fill_(7.0)
torch.cuda.synchronize()
t2 = bs[1].z_buffer()
print("zero-copy view:", float(t2[0].item()) == 7.0, t.data_ptr() == t2.data_ptr())
