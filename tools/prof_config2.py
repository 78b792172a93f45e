"""Config-2 fit, a few evaluations (profiling aid).  python tools/prof_config2.py [reps]"""
import sys
sys.path.insert(0, ".")
from paper_2603_16014_b200 import configs  # noqa: E402
from paper_2603_16014_b200.fast_gram import Model  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
inst = configs.make(2)
M = Model(inst.design)
M.set_y(inst.y)
for _ in range(reps):
    r = M.nll(inst.hyper, grad=True)
print("nll", r["nll"])
