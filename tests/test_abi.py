"""The C-ABI library loads on a CPU-only host, exports every symbol include/convpart.h
declares, and its host-only entry points (the partition planner, argument validation)
behave as specified (-m "not gpu"; no compute calls need a GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cpm():
    import __graft_entry__  # noqa: F401  (build on demand)
    from paper_1712_02546_b200 import build
    build.build()
    from paper_1712_02546_b200 import convpart
    convpart.lib()
    return convpart


def header_functions():
    src = open(os.path.join(ROOT, "include", "convpart.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(\w+)\s*\(", src, flags=re.M)))


def test_exports_every_declared_symbol(cpm):
    names = header_functions()
    assert len(names) >= 25
    lib = ctypes.CDLL(cpm.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), f"libconvpart.so does not export {n}"
    assert sorted(cpm.EXPORTS) == names


def test_planner_bitexact_vs_oracle(cpm, orc):
    g = np.random.default_rng(11)
    for _ in range(300):
        n = int(g.integers(1, 9))
        t = g.uniform(0.2, 7.0, n)
        k = int(g.integers(0, 4000))
        p = cpm.cp_partition_plan(list(t), k)
        kb, kc, kw = orc.plan(t, k)
        assert p.as_tuple() == (kb.tolist(), kc.tolist(), kw.tolist())
    np.testing.assert_allclose(cpm.cp_eq1_weights([10, 20, 40]), [4 / 7, 2 / 7, 1 / 7], rtol=1e-15)
    # the alignments the product uses: 32 (spanning N tiles) and 64 (bf16 operand mode, 64-element chunks)
    for align in (32, 64):
        for _ in range(100):
            n = int(g.integers(1, 9))
            t = g.uniform(0.2, 7.0, n)
            k = int(g.integers(0, 4000))
            p = cpm.cp_partition_plan(list(t), k, align)
            kb, kc, kw = orc.plan(t, k, align)
            assert p.as_tuple() == (kb.tolist(), kc.tolist(), kw.tolist())
            assert all(w % align == 0 and w >= c for w, c in zip(kw, kc))


def test_planner_errors(cpm):
    with pytest.raises(cpm.ConvPartError, match="CP_ERR_DATA"):
        cpm.cp_partition_plan([1.0, 0.0], 10)
    with pytest.raises(cpm.ConvPartError, match="CP_ERR_DATA"):
        cpm.cp_partition_plan([1.0, float("nan")], 10)
    with pytest.raises(cpm.ConvPartError, match="CP_ERR_CONFIG"):
        cpm.cp_partition_plan([], 10)
    with pytest.raises(cpm.ConvPartError, match="CP_ERR_ARG"):
        cpm.cp_partition_plan([1.0], -1)


def _desc(cpm, **kw):
    d = cpm.cp_conv_desc()
    d.batch, d.in_c, d.in_h, d.in_w, d.num_k, d.k_h, d.k_w = 4, 3, 32, 32, 8, 5, 5
    d.bias, d.relu, d.pool, d.math = 1, 1, 1, cpm.CP_MATH_FP32_SIMT
    d.input_kind = cpm.CP_INPUT_IMAGES
    d.out_part = cpm.cp_partition_plan([1.0], 8)
    d.rank, d.world = 0, 1
    for k, v in kw.items():
        setattr(d, k, v)
    return d


def test_create_validation(cpm):
    with pytest.raises(cpm.ConvPartError, match="CP_ERR_SHAPE.*dimension error"):
        cpm.conv_part_create(_desc(cpm, in_h=4))
    with pytest.raises(cpm.ConvPartError, match="CP_ERR_SHAPE.*pooling"):
        cpm.conv_part_create(_desc(cpm, in_h=31))
    with pytest.raises(cpm.ConvPartError, match="CP_ERR_SHAPE"):
        cpm.conv_part_create(_desc(cpm, num_k=9))
    with pytest.raises(cpm.ConvPartError, match="CP_ERR_CONFIG"):
        cpm.conv_part_create(_desc(cpm, rank=1))
    bad = cpm.cp_partition_plan([1.0, 1.0], 8)
    bad.k_width[0] = 3
    with pytest.raises(cpm.ConvPartError, match="CP_ERR_CONFIG"):
        cpm.conv_part_create(_desc(cpm, out_part=bad, world=2))


def test_product_path_has_no_oracle_dependency():
    """The product package never imports the oracle (no CPU fallback route)."""
    pkg = os.path.join(ROOT, "paper_1712_02546_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src).replace("oracle/", ""), f


def test_create_zero_kernel_ranks_host_side():
    """conv_part_create's host-side planning (validation, workspace sizing of all three passes) on
    partitions where a rank owns no kernels of a layer or an input block is empty: it must return a
    status (CP_OK on a GPU box, CP_ERR_CUDA where no device exists), never crash (a zero-width
    forward once divided by zero in the N-tile planner)."""
    from paper_1712_02546_b200 import convpart as cp
    for c1, c2 in [([36, 0], [40, 32]), ([12, 12, 12], [0, 72, 0]), ([0, 36], [72, 0])]:
        P = len(c1)
        p1, p2 = cp.cp_partition.from_counts(c1), cp.cp_partition.from_counts(c2)
        for r in range(P):
            for C, H, K, part, inp in [(3, 20, 36, p1, None), (36, 8, 72, p2, p1)]:
                for math in (cp.CP_MATH_TF32, cp.CP_MATH_FP32_SIMT):
                    d = cp.cp_conv_desc()
                    d.batch, d.in_c, d.in_h, d.in_w, d.num_k, d.k_h, d.k_w = 40, C, H, H, K, 5, 5
                    d.bias, d.relu, d.pool, d.math = 1, 1, 1, math
                    d.input_kind = cp.CP_INPUT_IMAGES if inp is None else cp.CP_INPUT_GATHER
                    d.out_part = part
                    if inp is not None:
                        d.in_part = inp
                    d.rank, d.world = r, P
                    try:
                        cp.conv_part_destroy(cp.conv_part_create(d, None))
                    except cp.ConvPartError as e:
                        assert e.rc == -5, str(e)     # CP_ERR_CUDA: no device here
