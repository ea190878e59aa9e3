"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package, and only as the checker.
The product package (paper_2503_18292_b200) never imports it.
"""
from .oracle import COracle, RefLib, c_oracle, ref_lib  # noqa: F401
