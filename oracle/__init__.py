"""TEST INFRASTRUCTURE ONLY — the DyLLM CPU oracle (NumPy, fp64).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this package. The product path
(`paper_2603_08026_b200`, `libdyllm.so`) never imports, links or executes it.
"""
from .dyllm_oracle import *  # noqa: F401,F403
