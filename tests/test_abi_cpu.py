"""CPU-side checks of the native boundary: the C-ABI library loads without a
GPU, exports every symbol include/glm_b200.h declares, and its host-only
entry points (xorshift jump, derive_seed) are bit-exact with the reference."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "glm_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(glm_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1803_06333_b200 import _lib
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_table_covers_header():
    from paper_1803_06333_b200 import _lib
    assert set(_declared()) == set(_lib.SIGNATURES)


def test_struct_layouts_match_header():
    from paper_1803_06333_b200 import _lib
    # glm_matrix: 3 x i64 + 2 x i32 + 4 pointers
    assert ctypes.sizeof(_lib.GlmMatrix) == 3 * 8 + 2 * 4 + 4 * 8
    # glm_solve_result: 6 x i32 + 3 x f64 + u64
    assert ctypes.sizeof(_lib.GlmSolveResult) == 6 * 4 + 3 * 8 + 8
    src = open(HEADER).read()
    body = src[src.index("typedef struct {\n    int32_t kind;"):src.index("} glm_solve_args;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"^\s+(?:const\s+)?\w+\s*\*?\s*(\w+);", body, flags=re.M)
    assert [f[0] for f in _lib.GlmSolveArgs._fields_] == fields


def test_host_jump_and_derive_seed_bit_exact(lib, golden):
    z = golden("prng")
    for c, (seed, n) in enumerate(z["perm_cases"]):
        states = [int(x) for x in z[f"perm{c}_states"]]
        assert lib.glm_xorshift_jump(states[0], int(n)) == states[1]
        assert lib.glm_xorshift_jump(states[0], 2 * int(n)) == states[2]
    for i, s in enumerate(z["derive1_seeds"]):
        for j, ix in enumerate(z["derive1_idx"]):
            arr = np.array([int(ix)], dtype=np.uint64)
            got = lib.glm_derive_seed(int(s), arr.ctypes.data_as(ctypes.c_void_p), 1)
            assert got == int(z["derive1"][i, j])


def test_last_error_is_a_string(lib):
    from paper_1803_06333_b200 import _lib
    assert isinstance(_lib.last_error(), str)


def test_python_mirror_prng_matches_reference(golden):
    import paper_1803_06333_b200 as g
    z = golden("prng")
    assert g.derive_seed(13, 0) == 0xBC10FE74B44B54C8
    for i, s in enumerate(z["derive1_seeds"]):
        assert g.solver.splitmix64(int(s)) == int(z["splitmix"][i])
    gen = g.PermutationGenerator(5)
    gen.advance(3)
    st = 5
    for _ in range(3):
        st = g.solver.xorshift64_step(st)
    assert gen.state == st
