"""CPU oracle for the MR-GPTQ quantized-linear hot path (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU reference.  The product package ``paper_2509_23202_b200`` never
imports it and has no CPU fallback.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference
(``/root/reference/pkg/src/microfp``) in the dev container and commits its
outputs under ``tests/golden/``; ``tests/test_oracle.py`` checks this
restatement against those fixtures and against the reference's own golden
SHA-256 container hashes (``pkg/tests/test_acceptance.py:335-361``).
"""

from .microfp_oracle import *  # noqa: F401,F403
from .microfp_oracle import __all__  # noqa: F401
