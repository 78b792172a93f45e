"""Where does a config-2 fit's wall time go?  Development aid (prints only).
python tools/latency_probe.py [config]"""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_16014_b200 import configs  # noqa: E402
from paper_2603_16014_b200._lib import CResult  # noqa: E402
from paper_2603_16014_b200.fast_gram import Model  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
inst = configs.make(cfg)
M = Model(inst.design)
M.set_y(inst.y)
hp = inst.hyper
stream = torch.cuda.ExternalStream(M.stream, device=torch.device("cuda", 0))
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")
for _ in range(5):
    M.nll(hp)


def ev_loop(n, prof, do_flush):
    M.profile(prof)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    torch.cuda.synchronize()
    for k in range(n):
        if do_flush:
            with torch.cuda.stream(stream):
                flush.fill_(float(k))
        ev[k][0].record(stream)
        M.nll(hp)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    p = M.profile_read() if prof else {}
    M.profile(False)
    return 1e3 * sum(a.elapsed_time(b) for a, b in ev) / n, {k: 1e3 * v[0] / max(v[1], 1) for k, v in p.items()}


for prof in (True, False):
    for fl in (True, False):
        us, ks = ev_loop(200, prof, fl)
        print(f"events/step prof={prof} flush={fl}: {us:.1f} us  kernels {ks}  sum {sum(ks.values()):.1f}")

ch = M._hyper_struct(hp)
r = CResult()
lib, h = M.lib, M.h
for name, fn in (("raw ctypes fmtgp_nll", lambda: lib.fmtgp_nll(h, C.byref(ch), 1, C.byref(r))),
                 ("Model.nll", lambda: M.nll(hp))):
    for _ in range(20):
        fn()
    t = time.perf_counter()
    for _ in range(1000):
        fn()
    print(f"wall/step {name}: {(time.perf_counter() - t) * 1e3:.1f} us")

# ---- end to end: pinned y -> set_y -> nll (as bench.py's e2e), split
M = Model(inst.design)
M.set_y(inst.y)
stream = torch.cuda.ExternalStream(M.stream, device=torch.device("cuda", 0))
y_pinned = torch.empty(inst.design.N, dtype=torch.float64).pin_memory().numpy()
y_pinned[:] = inst.y
for _ in range(5):
    M.set_y(y_pinned)
    M.nll(hp)
for what in ("set_y", "set_y+nll"):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(100):
        with torch.cuda.stream(stream):
            flush.fill_(float(k))
        ev[k][0].record(stream)
        M.set_y(y_pinned)
        if what != "set_y":
            M.nll(hp)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    print(f"e2e events/step {what}: {1e3 * sum(a.elapsed_time(b) for a, b in ev) / 100:.1f} us")
t = time.perf_counter()
for _ in range(200):
    lib.fmtgp_model_set_y(M.h, y_pinned.ctypes.data_as(C.POINTER(C.c_double)))
print(f"wall/step raw set_y pinned: {(time.perf_counter() - t) * 1e6 / 200:.1f} us")
t = time.perf_counter()
for _ in range(200):
    lib.fmtgp_model_set_y(M.h, inst.y.ctypes.data_as(C.POINTER(C.c_double)))
print(f"wall/step raw set_y pageable: {(time.perf_counter() - t) * 1e6 / 200:.1f} us")
M.close()
