"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the DG operator path.

Nothing in the product package (``paper_1403_1157_b200``) may import
this package.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` legs use it, and only
as the checker or the timed CPU reference arm.

Parity status: PINNED.  ``tests/test_oracle_golden.py`` checks this
restatement against fixtures produced by running the real reference
(``tests/golden/make_golden.py`` imports ``taxisdg`` from
/root/reference and calls its public API).
"""

from .taxis_oracle import (OracleOperator, ssprk3, bump_field,  # noqa: F401
                           sdirk_integrate)
