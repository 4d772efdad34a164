import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, agcn_inputs as gen, paper_2308_11825_b200 as A
for c in ("c1", "c2"):
    w = gen.make_config(c)
    rp = torch.from_numpy(w.rowptr).cuda(); ci = torch.from_numpy(w.colidx).cuda()
    for _ in range(3):
        A.Plan(rp, ci, max_block_warps=0, max_warp_nzs=0).close()
    torch.cuda.synchronize()
