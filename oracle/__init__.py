"""fp64 CPU oracle (test infrastructure only; see oracle/tilt_oracle.py header)."""
from .tilt_oracle import *  # noqa: F401,F403
