"""CPU parity oracle for the B200 GLM hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu-baseline /
`--impl reference` leg may import this package. The product package
`paper_1803_06333_b200` never imports it, and its CUDA path fails loudly when
its own extension is missing instead of falling back here.

`oracle.core` restates the reference (`hierglm`, /root/reference/pkg/src) in C
(`glm_oracle.c`, loaded through ctypes) plus numpy for the O(d) engine glue;
every function cites the reference file:line it follows. Parity of the oracle
itself is pinned against `tests/golden/*.npz`, produced by running the
reference (`tests/golden/make_golden.py`).
"""

from .core import *  # noqa: F401,F403
