import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, ctypes
import agcn_inputs as gen, paper_2308_11825_b200 as A
from paper_2308_11825_b200 import _lib
L = _lib.lib()
w = gen.make_config("c1")
rp = torch.from_numpy(w.rowptr).cuda(); ci = torch.from_numpy(w.colidx).cuda()
o = _lib.Opts(); L.agcn_default_opts(ctypes.byref(o))
for _ in range(20):
    h = L.agcn_plan_ex(rp.data_ptr(), ci.data_ptr(), w.n, w.nnz, ctypes.byref(o)); L.agcn_plan_destroy(h)
torch.cuda.synchronize()
ts = []
for _ in range(200):
    t0 = time.perf_counter()
    h = L.agcn_plan_ex(rp.data_ptr(), ci.data_ptr(), w.n, w.nnz, ctypes.byref(o))
    t1 = time.perf_counter()
    L.agcn_plan_destroy(h)
    ts.append(t1 - t0)
ts.sort()
print("agcn_plan_ex host wall (C1): median %.1f us, p10 %.1f us" % (1e6 * ts[100], 1e6 * ts[20]))
ts = []
for _ in range(200):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = A.Plan(rp, ci)
    t1 = time.perf_counter()
    p.close()
    ts.append(t1 - t0)
ts.sort()
print("A.Plan python wall (C1): median %.1f us" % (1e6 * ts[100]))
