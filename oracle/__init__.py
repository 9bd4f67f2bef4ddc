"""CPU oracle for the DSV dynamic-sparsity attention path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithms (reference package
`dynsparse`, /root/reference/pkg/src/dynsparse), each function citing the
reference file:line it follows. It is the checker for the CUDA path:
only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import it. The product path (paper_2502_07590_b200) never
imports or calls anything here.

Parity pinning: tests/test_oracle_golden.py checks every function here against
golden vectors produced by running the reference itself
(tests/golden/make_golden.py imports /root/reference in the build container and
writes tests/golden/*.npz). The sparse-attention backward has no reference
test; its golden vectors come from the reference's own autograd formulation
(`_Block.attention`, pkg/src/dynsparse/trainer.py:104-118) run by that script.
"""

from .selection import k_from_sparsity, topk_from_scores, topk_lowrank  # noqa: F401
from .attention import (  # noqa: F401
    full_attention,
    grouped_attention_fwd,
    grouped_attention_bwd,
    rows_attention_fwd,
    rows_attention_bwd,
)
from .grouping import build_groups  # noqa: F401
