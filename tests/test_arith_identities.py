"""Arithmetic identities the kernels rely on for bit-exactness, checked in exact rational
arithmetic (no GPU, no oracle).

Markstein division (the LIST kernel's exact means, eval.cu): with r = RN(1/n), q0 = RN(S r),
e = RN(S - n q0) and q = RN(q0 + e r), q == RN(S / n) for integer S < 2^41 (sums of at most
512 Q32 values) and 1 <= n <= 512 (LIST divides by V; the wider n range covers any stream
count up to 512).  Each RN(.) below is one IEEE binary64 operation with a
single rounding (Fraction -> float is correctly rounded), exactly what DMUL / DFMA do."""
import random
from fractions import Fraction as F


def _rn(x):
    return float(x)


def test_markstein_division_exact_for_kernel_ranges():
    rng = random.Random(20121)
    checked = 0
    for n in range(1, 513):
        r = _rn(F(1, n))
        samples = [rng.randrange(0, 2**41) for _ in range(24)]
        samples += [k * n + d for k in (1, 3, 2**20 // n, 2**30 // n, 2**40 // n) for d in (-1, 0, 1)
                    if 0 <= k * n + d < 2**41]
        samples += [2**41 - 1, (2**41 // n) * n, 2**40 + 1, 0, 1]
        for S in samples:
            a = float(S)
            q0 = _rn(F(a) * F(r))
            e = _rn(-F(n) * F(q0) + F(a))
            q = _rn(F(e) * F(r) + F(q0))
            assert q == _rn(F(S, n)), (S, n)
            checked += 1
    assert checked > 10000
