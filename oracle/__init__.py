"""CPU oracle for the EvConv incremental path -- TEST INFRASTRUCTURE ONLY.

This package is the *checker*, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
(``cpu_baseline`` / ``--impl reference``) may import it.  The product
package ``paper_2303_04670_b200`` never imports anything from here and
fails loudly when its CUDA library is missing.

``evincr_np`` restates the reference package ``evincr`` 0.1.0
(``/root/reference/pkg/src/evincr``) in numpy; each function cites the
reference file:line it follows.

Parity pinning: the restatement is checked against golden vectors that
``tests/golden/make_golden.py`` produced by importing the real reference
in the build container (``tests/test_oracle_golden.py``).
"""
