# Per-warp trace of one C2 walk (tp_debug_trace): SM id, start/end clock, items.
# Run on a B200: python tools/trace_warps.py
import sys, os, json, numpy as np, torch, ctypes
sys.path.insert(0, '.')
from paper_2407_20205_b200 import _kernels, fixtures
n, B = 24, 16384
e = torch.from_numpy(fixtures.uniform_batch(n, 0, 0, B)).cuda()
rows = torch.empty((B, 2048), dtype=torch.uint8, device='cuda')
pm = torch.zeros((B, 2), dtype=torch.int64, device='cuda')
tr = torch.zeros((148 * 64 * 4, 4), dtype=torch.int64, device='cuda')
st = torch.cuda.current_stream().cuda_stream
_kernels.pack_async(e.data_ptr(), B, n, rows.data_ptr(), st)
_kernels.walk_async(rows.data_ptr(), B, n, pm.data_ptr(), st)
torch.cuda.synchronize()
_kernels.lib().tp_debug_trace(ctypes.c_void_p(tr.data_ptr()))
pm.zero_()
_kernels.walk_async(rows.data_ptr(), B, n, pm.data_ptr(), st)
torch.cuda.synchronize()
t = tr.cpu().numpy()
t = t[t[:, 3] > 0]
sm = t[:, 0]; s0 = t[:, 1]; s1 = t[:, 2]; it = t[:, 3]
print("warps traced", len(t), "items min/max", it.min(), it.max())
cnt = np.bincount(sm, minlength=148)
print("CTAs per SM: min", cnt.min(), "max", cnt.max(), "hist", np.bincount(cnt))
dur = (s1 - s0)
print("duration cycles: min %.3e median %.3e max %.3e" % (dur.min(), np.median(dur), dur.max()))
for q in (0, 1, 2, 100):
    m = sm == q
    print("sm", q, "ctas", m.sum(), "start spread", s0[m].max() - s0[m].min(), "end spread", s1[m].max() - s1[m].min(), "dur med", np.median(dur[m]), "min", dur[m].min(), "max", dur[m].max())
