"""Phase timeline of the fused digital fit (FMTGP_TRACE=1 globaltimer marks, printed by the
library to stderr), with an L2 flush before each evaluation as in bench.py.
python tools/trace_config2.py [reps]"""
import os
import sys

os.environ["FMTGP_TRACE"] = "1"
sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2603_16014_b200 import configs  # noqa: E402
from paper_2603_16014_b200.fast_gram import Model  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 3
inst = configs.make(2)
M = Model(inst.design)
M.set_y(inst.y)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")
for k in range(reps):
    if "--no-flush" not in sys.argv:
        flush.fill_(float(k))
    torch.cuda.synchronize()
    print(f"--- eval {k}", file=sys.stderr, flush=True)
    M.nll(inst.hyper, grad=True)
