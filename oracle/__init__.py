"""TEST INFRASTRUCTURE — CPU oracle for the slab-Ewald solve.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / the timed reference
arm.  The product (``paper_2101_07088_b200``) never imports it; its solve
path runs on the GPU and fails loudly without the CUDA library.

Parity status: PINNED.  ``tests/golden/make_golden.py`` ran the reference
package (``slabewald`` 0.1.0 from ``/root/reference/pkg/src``) in the build
container and stored its outputs under ``tests/golden/``;
``tests/test_oracle_golden.py`` checks this restatement against them.
"""

from .slab_oracle import OracleSlabSolver, oracle_solve  # noqa: F401
