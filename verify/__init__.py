"""GPU-side result checkers for full-size parity (sortedness + multiset
digest).  Test/bench infrastructure, not part of the sort."""
from .verify import sorted_check, digest  # noqa: F401
