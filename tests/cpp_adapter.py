"""Build + drive tests/cpp/adapter_check.cpp (the C++ adapter over the C ABI)."""
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "adapter_check.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "adapter_check")
LIBDIR = os.path.join(ROOT, "paper_2603_16014_b200")


def build():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < max(os.path.getmtime(SRC), os.path.getmtime(
            os.path.join(ROOT, "include", "fastmtgp_b200.hpp"))):
        subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), SRC, "-o", BIN,
                        f"-L{LIBDIR}", "-l:libfmtgp_b200.so", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return BIN


def serialize(dz, hp, R, y):
    parts = [dz.kind, dz.d, dz.L, *dz.m]
    if dz.kind == 0:
        parts += [dz.n_max, *[int(v) for v in dz.g]]
    else:
        parts += [dz.columns.shape[1], *[int(v) for v in dz.columns.ravel()]]
    parts += [int(v) for v in dz.shift_bits.ravel()]
    parts += [repr(float(hp.gamma)), hp.si_alpha, *[repr(float(v)) for v in hp.b], *[repr(float(v)) for v in hp.eta]]
    parts += [repr(float(v)) for v in np.asarray(R).ravel()] + [repr(float(v)) for v in hp.xi]
    parts += [len(y)] + [repr(float(v)) for v in y]
    return " ".join(str(p) for p in parts)


def run(dz, hp, R, y):
    p = subprocess.run([build()], input=serialize(dz, hp, R, y), capture_output=True, text=True)
    out = {"rc": p.returncode, "stderr": p.stderr}
    if p.returncode == 0:
        lines = p.stdout.split("\n")
        out["logdet"] = float(lines[0].split()[1])
        out["x"] = np.array([float(v) for v in lines[1].split()[1:]])
    return out
