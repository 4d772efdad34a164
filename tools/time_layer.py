"""Time one GCN layer (paper_2308_11825_b200.layer.GCNLayer: tcgen05 X.W + agcn SpMM with the
fused bias/ReLU epilogue) on a config, and its X.W alone (libagcn at the layer's precision, and
cuBLAS fp32 for comparison): python tools/time_layer.py c5 64 64 [fp32|tf32]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import agcn_inputs as gen  # noqa: E402
import paper_2308_11825_b200 as A  # noqa: E402
from paper_2308_11825_b200.layer import GCNLayer  # noqa: E402

name, fin, fout = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
prec = sys.argv[4] if len(sys.argv) > 4 else "fp32"
w = gen.make_config(name)
dev = torch.device("cuda:0")
rp, ci, va = (torch.from_numpy(a).to(dev) for a in (w.rowptr, w.colidx, w.vals))
X = torch.from_numpy(w.X(fin)).to(dev)
g = torch.Generator(device="cpu").manual_seed(0)
W = (torch.rand((fin, fout), generator=g) - 0.5).to(dev)
b = (torch.rand(fout, generator=g) - 0.5).to(dev)
plan = A.Plan(rp, ci)
layer = GCNLayer(plan, va, W, b, relu=True, precision=prec)
for _ in range(3):
    Y = layer(X)
torch.cuda.synchronize()
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
e0, e1 = ev(), ev()
e0.record()
for _ in range(10):
    Y = layer(X)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
torch.backends.cuda.matmul.allow_tf32 = False
Wt = W.t().contiguous()
e0.record()
for _ in range(10):
    T = A.gemm_xw(X, Wt, precision=prec)
e1.record()
torch.cuda.synchronize()
gemm = e0.elapsed_time(e1) / 10
e0.record()
for _ in range(10):
    T = torch.mm(X, W)
e1.record()
torch.cuda.synchronize()
cub = e0.elapsed_time(e1) / 10
gb = 4.0 * w.n * (fin + fout) / 1e9
print(json.dumps({"config": name, "fin": fin, "fout": fout, "precision": prec, "order": layer.order, "layer_ms": ms,
                  "gemm_XW_ms": gemm, "gemm_XW_TBps": gb / gemm, "cublas_fp32_XW_ms": cub,
                  "flops": 2 * w.nnz * min(fin, fout) + 2 * w.n * fin * fout}))
