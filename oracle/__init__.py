"""CPU oracle for the Logits-Cache re-sampling path -- TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the reference algorithms that the CUDA
path replaces (``/root/reference/pkg/src/agentserve``; every function cites
the file:line it follows).  It exists to *check* the product, never to be
the product:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2604_17353_b200`` never imports it and has no
  CPU fallback (it raises if its CUDA library is missing).

Parity pinning: the restatement is checked against golden vectors produced
by importing the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz|json``) and against
the reference's own known-answer tests.
"""
