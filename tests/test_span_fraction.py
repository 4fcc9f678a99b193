"""MaxMin's span in the TMEM tier (R-6): span = floor((hi - lo) u^3 / T^3)
with u = T - t is computed from a per-step 64-bit fraction f_t = floor(2^64 u^3 / T^3)
(runtime.cu, the `mtab` table) as est = floor(a f_t / 2^64), then one remainder
test (a u^3 - est T^3 >= T^3 -> est + 1; tmem_kernel.cuh).  The claim that this
is exactly the floor for every a < 2^32 and T <= 65536 rests on the bound
est >= floor(a u^3/T^3) - 1 (a f_t / 2^64 > a u^3/T^3 - a / 2^64 > x - 2^-32).
This pins the arithmetic against Python's exact integers, including the
extremes; the GPU parity tests pin the kernel that uses it."""
import random

import pytest


def span_by_fraction(a: int, t: int, T: int) -> int:
    u = T - t
    f = ((u ** 3) << 64) // (T ** 3)            # the host table entry (u^3 < T^3, so f < 2^64)
    assert 0 <= f < 1 << 64
    est = (a * f) >> 64                         # __umul64hi
    q = T ** 3
    rem = (a * u ** 3 - est * q) % (1 << 64)    # wrapping 64-bit arithmetic, as on the device
    if rem >= q:
        est += 1
    return est


@pytest.mark.parametrize("T", [1, 2, 3, 7, 100, 3277, 65535, 65536])
def test_span_extremes(T):
    for a in (0, 1, 2, 255, (1 << 31) - 1, (1 << 32) - 1):
        for t in {tt for tt in (1, 2, T // 2, T - 1, T) if 1 <= tt <= T}:
            assert span_by_fraction(a, t, T) == a * (T - t) ** 3 // T ** 3, (a, t, T)


def test_span_random():
    rng = random.Random(2207)
    for _ in range(20000):
        T = rng.choice([rng.randint(1, 65536), rng.randint(1, 5000), 3277])
        t = rng.randint(1, T)
        a = rng.randrange(1 << 32)
        assert span_by_fraction(a, t, T) == a * (T - t) ** 3 // T ** 3, (a, t, T)


def test_span_near_integer_boundaries():
    """a u^3 / T^3 just below an integer is where a one-step estimate can be off."""
    rng = random.Random(7)
    hits = 0
    for _ in range(20000):
        T = rng.randint(2, 65536)
        t = rng.randint(1, T - 1)
        u3, q = (T - t) ** 3, T ** 3
        k = rng.randint(1, 1 << 20)
        a = (k * q) // u3                        # a u^3 / T^3 just below (or at) the integer k
        if a >= 1 << 32:
            continue
        hits += 1
        for da in (-1, 0, 1):
            aa = a + da
            if 0 <= aa < 1 << 32:
                assert span_by_fraction(aa, t, T) == aa * u3 // q
    assert hits > 1000
