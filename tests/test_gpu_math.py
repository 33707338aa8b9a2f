"""The kernels' slow-path-free IEEE rcp / div / sqrt equal CUDA's library operators bit for bit."""
import pytest

pytestmark = pytest.mark.gpu


def test_ieee_ops_bitwise(gpu):
    from paper_1307_4839_b200.swof import selftest_math
    for seed in (1, 1307, 2 ** 40 + 7):
        assert selftest_math(1 << 24, seed) == (0, 0, 0)
