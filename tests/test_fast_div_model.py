"""The kernels' thread-group arithmetic divides small non-negative integers
with a float reciprocal (csrc/hmx_kernels.cu fast_div: int((a + 0.5f) *
rcp_rn(b))).  Model it in float32 and check it against integer division over
the whole range the kernels use (a <= 2048 * 257, 1 <= b <= 256)."""
import numpy as np


def fast_div(a, b):
    r = (np.float32(1.0) / b.astype(np.float32)).astype(np.float32)      # __frcp_rn
    return ((a.astype(np.float32) + np.float32(0.5)) * r).astype(np.float32).astype(np.int64)


def test_fast_div_is_exact_over_the_kernel_range():
    a = np.arange(0, 2048 * 257 + 1, dtype=np.int64)
    for b in range(1, 257):
        q = fast_div(a, np.full_like(a, b))
        assert np.array_equal(q, a // b), b
