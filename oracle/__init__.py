"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the polynomial-filtering hot path.

* ``oracle.clib``   -- ctypes view of the plain-C restatement (``oracle/sliceeig_oracle.c``).
* ``oracle.reflib`` -- ctypes view of the unmodified reference compiled in place
  (``oracle/_ref/libsliceeig_ref.so`` built from ``/root/reference/proj/include`` by
  ``oracle/Makefile``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference/cpu_baseline legs may
import this package, and only as the checker / the timed CPU baseline.  The product package
``paper_1802_05215_b200`` never imports it.
"""
