"""CPU oracle for the trajectory-manager hot path — TEST INFRASTRUCTURE ONLY.

* ``oracle/radix.py``        pure-Python restatement of the reference SessionTrie
                             (small cases; pinned to tests/golden by
                             tests/test_oracle_golden.py).
* ``oracle/radix_oracle.c``  the same algorithm in C (large cases and the CPU
                             baseline timed by bench.py), pinned to radix.py and
                             the golden vectors by tests/test_oracle_c.py.
* ``oracle/cport.py``        ctypes loader for the C restatement.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package, and only as the checker or the timed CPU
reference.  The product package never imports it.
"""
