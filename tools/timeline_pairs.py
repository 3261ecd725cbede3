import os, sys
sys.path.insert(0, "/root/repo")
os.environ["SR_TIMELINE"] = "1"
import numpy as np, torch
import paper_1609_04471_b200 as sr
from workloads import gen
n = 16777216
k = torch.from_numpy(gen.make("few100", n, np.int32, config=3)).cuda()
v = torch.arange(n, dtype=torch.int32, device="cuda")
wk, wv = torch.empty_like(k), torch.empty_like(v)
for i in range(3):
    wk.copy_(k); wv.copy_(v); torch.cuda.synchronize(); sr.sort_pairs(wk, wv); torch.cuda.synchronize()
sr.set_option(sr.OPT_PROFILE, 1)
wk.copy_(k); wv.copy_(v); torch.cuda.synchronize(); sr.sort_pairs(wk, wv); torch.cuda.synchronize()
print(sr.last_plan(), file=sys.stderr)
