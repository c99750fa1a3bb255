"""ORACLE -- TEST INFRASTRUCTURE ONLY.

CPU restatement of the reference package ``topovox`` (Python/numba, not
importable on the GPU box) used as the parity checker by ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py``. Nothing in ``paper_2203_15115_b200`` imports this
package; the product path is CUDA-only and fails loudly without its library.

Pinning: the restatement is checked against golden vectors produced by the
real reference in the build container (``tests/golden/make_golden.py``) and
against the SPEC's known-answer examples (``tests/test_oracle.py``).
"""
