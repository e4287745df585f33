"""fp64 CPU oracle of the AutoFreeze freezing hot path -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything under `oracle/`.
The product package `paper_2102_01386_b200` never imports it and has no CPU
fallback; the two share no code (only the seeded generators in `afinputs/`).
"""
from .autofreeze_oracle import *  # noqa: F401,F403
from .autofreeze_oracle import __all__  # noqa: F401
