"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO simulation or placement-search arithmetic: it only
builds the inputs both sides consume -- model/config tables (Table 1 of the
paper, plus the stage-partition planner of §4.1) and
time-sorted int64-nanosecond request traces (Gamma renewal arrivals, §5.2
P:100; power-law per-model splits, §5.3).  Both `oracle/` and
`paper_2302_11665_b200/` may import it; it imports neither.

Citations: `P:n` = line n of the paper text, `S:n` = line n of
the CPU-program spec, used for interfaces only.
"""

from .problem import Problem, Trace, Placement  # noqa: F401
from . import table1, planner, traces, configs  # noqa: F401
