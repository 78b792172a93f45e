"""Larger seeded random-shape sweep of the fused lattice path and its sharding (60 cases; the
test suite runs 12 of the same generator).  python tools/sweep_lattice_fused.py"""
import sys
sys.path.insert(0, ".")
import tests.test_gpu_lattice_fused as t
cases = t._random_cases(60, seed=777)
bad = 0
for c in cases:
    try:
        t.test_fused_random_shapes(c)
    except Exception as e:
        bad += 1
        print("FAIL", c, repr(e)[:300])
print("done", len(cases), "bad", bad)
