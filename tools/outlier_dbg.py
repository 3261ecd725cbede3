import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_04471_b200 as sr
from workloads import gen
for n, k in [(100003, 1), (100003, 10), (2_000_000, 20000)]:
    a = gen.swaps(n, k, np.int32, 1000 + k)
    d = torch.from_numpy(a.copy()).cuda()
    sr.sort_keys(d); torch.cuda.synchronize()
    print(n, k, sr.last_plan(), bool((d.cpu().numpy() == np.sort(a)).all()), file=sys.stderr)
    # where are the descents of the input?
    desc = np.nonzero(a[:-1] > a[1:])[0]
    print("descents at", desc[:10], file=sys.stderr)
