"""CPU oracle for the adaptive H^2 x H^2 product (TEST INFRASTRUCTURE ONLY).

This package restates, in plain NumPy, the algorithm of the reference
package ``h2mul`` (arXiv 2309.09061) for the path this repository
accelerates: ``multiply`` (phase 1) followed by ``coarsen`` (phase 2).
Every function cites the reference file:line it follows.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline legs may import it, and only as the checker / the timed CPU
baseline.  The GPU product path never routes through it.

Pinning: ``tests/test_oracle_golden.py`` checks this restatement against
golden vectors produced by the reference itself
(``tests/golden/make_golden.py``, run in the build container where
``/root/reference`` is importable).
"""

from .h2_oracle import *  # noqa: F401,F403
