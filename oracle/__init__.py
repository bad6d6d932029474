"""CPU oracle for the TFLMS executor path — TEST INFRASTRUCTURE ONLY.

Restatements of the reference's CPU executor (``interp.py``) and of its
memory/transfer model (``sim.py``), pinned against golden vectors that the
reference itself produced (tests/golden/make_golden.py).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / reference leg
may import this package, and only as the checker or the timed CPU baseline;
the product path (``paper_1807_02037_b200``) never imports it.
"""
