"""CPU oracle for the IsoQuant stage-1 path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
--impl reference arm) may import this package.  See iq_oracle.py."""
from . import iq_oracle  # noqa: F401
