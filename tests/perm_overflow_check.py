"""Run under GLM_PERM_REGION_CAP=<small> (tests/test_gpu_solver.py): every
bucket outgrows its region, so the permutations come from the overflow lists
and the slow path; they must equal the oracle's stable argsort bit for bit."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1803_06333_b200 as g  # noqa: E402
from paper_1803_06333_b200 import pipeline  # noqa: E402

assert os.environ.get("GLM_PERM_REGION_CAP"), "set GLM_PERM_REGION_CAP"
for seed, n in [(5, 3), (7, 4095), (11, 70_001), (13, 300_007)]:
    gen = g.PermutationGenerator(seed)
    got = gen.permute(n)
    want, st = oracle.permute(seed, n)
    np.testing.assert_array_equal(got, want)
    assert gen.state == st
    np.testing.assert_array_equal(pipeline.chunk_permutation(seed, n),
                                  oracle.argsort_stable(oracle.generate_keys(seed, n)))
print("overflow path ok")
