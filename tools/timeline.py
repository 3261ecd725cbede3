import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SR_TIMELINE"] = "1"
import numpy as np, torch
import paper_1609_04471_b200 as sr
from workloads import gen
n = int(sys.argv[1]); order = sys.argv[2] if len(sys.argv) > 2 else "random"
dt = np.int64 if (len(sys.argv) > 3 and sys.argv[3] == "i64") else np.int32
src = torch.from_numpy(gen.make(order, n, dt, config=4)).cuda()
w = torch.empty_like(src)
for i in range(3):
    w.copy_(src); torch.cuda.synchronize(); sr.sort_keys(w); torch.cuda.synchronize()
sr.set_option(sr.OPT_PROFILE, 1)
w.copy_(src); torch.cuda.synchronize(); sr.sort_keys(w); torch.cuda.synchronize()
print(sr.last_plan(), file=sys.stderr)
