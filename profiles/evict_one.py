"""A few evict_select calls on the `evict` config (for ncu: -k regex:evict_select)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_03651_b200 as K  # noqa: E402
import workloads as W  # noqa: E402

if "--ctas" in sys.argv:
    K.set_option("evict_ctas", int(sys.argv[sys.argv.index("--ctas") + 1]))
dev = torch.device("cuda", 0)
ev = W.make_evict(straddle="straddle" in sys.argv)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(dev)  # noqa: E731
keys = K.evict_keys(t(ev.state, np.uint8), t(ev.rc, np.int32), t(ev.lat, np.int32), t(ev.depth, np.int16))
ws = torch.zeros(K.evict_select_workspace_size(len(ev.state), ev.k), dtype=torch.uint8, device=dev)
ids = torch.empty(ev.k, dtype=torch.int32, device=dev)
for _ in range(3):
    K.evict_select(keys, ev.k, out_ids=ids, workspace=ws, sync=False)
torch.cuda.synchronize()
print("ok")
