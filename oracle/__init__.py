"""TEST INFRASTRUCTURE ONLY: the CPU oracle for the A^k hot path.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference legs, where it is the checker (never the thing
measured as the product).  See oracle/oracle.py for the restatement and
oracle/matexpo_oracle.c for the C core.  Parity status: pinned against
tests/golden (generated from the unmodified reference).
"""

from .oracle import *  # noqa: F401,F403
from .oracle import __all__  # noqa: F401
