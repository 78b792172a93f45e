"""CPU oracle (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package, and only as the checker or the CPU baseline — never
as the thing measured or shipped.  The product (paper_2603_16014_b200) never
imports it and fails loudly when its CUDA library is missing.

* ``oracle.ref``  — the reference C++ library itself (oracle/_ref, built by
  oracle/Makefile from /root/reference/proj/src with our Eigen-subset shim).
* ``oracle.port`` — our C restatement (oracle/fmtgp_oracle.c), each function
  citing the reference file:line it follows; pinned against the reference's own
  known-answer tests and against golden vectors generated from oracle.ref
  (tests/golden/, scripts/make_golden.py).
"""
