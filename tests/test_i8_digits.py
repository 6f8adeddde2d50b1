"""The fixed-point format of the int8 M2L (csrc/k_m2l_i8.cu, kernels.hpp), restated in
numpy and checked on the CPU: balanced base-256 digits, the scale rule, the kept
digit pairs and the int32 accumulator bound.  The GPU tests check the kernel itself
against the oracle; this file pins the arithmetic the kernel relies on."""
import numpy as np
import pytest

KS, BITS, LEVELS = 6, 8, 7  # kI8Digits, kI8Bits, kI8Levels defaults (kernels.hpp)


def level_exp(mx):
    """Exponent ex of the scale S = 2^(ex + 1): frexp of the maximum bumped by 2^-6."""
    return int(np.frexp(mx * 1.015625)[1])


def to_digits(x, ex):
    """x -> KS balanced base-2^BITS digits, most significant first (k_m2l_i8.cu to_digits)."""
    h = 1 << (BITS - 1)
    X = np.rint(np.ldexp(x, BITS * KS - ex - 1)).astype(np.int64)
    d = np.zeros((KS,) + x.shape, dtype=np.int64)
    for i in range(KS - 1, 0, -1):
        r = ((X + h) & (2 * h - 1)) - h
        d[i] = r
        X = (X - r) >> BITS
    d[0] = X
    return d


def from_digits(d, ex):
    acc = np.zeros(d.shape[1:], dtype=np.float64)
    for i in range(KS - 1, -1, -1):
        acc += np.ldexp(d[i].astype(np.float64), -BITS * (i + 1))
    return np.ldexp(acc, ex + 1)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_digits_fit_int8_and_reconstruct(seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(20000) * 10.0 ** rng.uniform(-6, 0, 20000)
    # adversarial maxima: just below / at / above a power of two
    for mx in (1.0 - 2.0 ** -50, 1.0, 1.0 + 2.0 ** -40, 0.75, 0.5000001):
        v = np.concatenate([x / np.abs(x).max() * mx, [mx, -mx]])
        ex = level_exp(np.abs(v).max())
        d = to_digits(v, ex)
        assert d.min() >= -128 and d.max() <= 127  # every digit is an int8
        err = np.abs(from_digits(d, ex) - v).max()
        assert err <= np.ldexp(1.0, ex + 1 - BITS * KS - 1) * (1 + 1e-9)  # half an ulp of 48 bits of S
    # the negated imaginary part has its own digits: the same value with the sign flipped
    ex = level_exp(np.abs(x).max())
    assert np.array_equal(from_digits(to_digits(-x, ex), ex), -from_digits(to_digits(x, ex), ex))


def test_truncated_digit_product_error():
    """sum over the kept pairs i + j <= LEVELS - 1 vs the exact product of the rounded
    operands: the dropped pairs weigh <= 2^(-BITS (LEVELS + 2)) 128^2 each."""
    rng = np.random.default_rng(5)
    K = 704
    w = rng.uniform(-1, 1, (64, K))
    v = rng.uniform(-1, 1, K)
    ew, ev = level_exp(np.abs(w).max()), level_exp(np.abs(v).max())
    dw, dv = to_digits(w, ew), to_digits(v, ev)
    acc = np.zeros((LEVELS, 64), dtype=np.int64)
    for i in range(KS):
        for j in range(KS):
            if i + j <= LEVELS - 1:
                acc[i + j] += dw[i] @ dv[j]
    assert np.abs(acc).max() < 2 ** 31 // 31  # 31 keys of this K fit an int32 accumulator
    got = sum(np.ldexp(acc[L].astype(np.float64), -BITS * (L + 2)) for L in range(LEVELS - 1, -1, -1))
    got = np.ldexp(got, ew + ev + 2)
    ref = w @ v
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel < 2e-14, rel
    # without the level-6 pairs (21 products) the truncation dominates: ~6x larger
    acc6 = acc[: LEVELS - 1]
    got6 = np.ldexp(sum(np.ldexp(acc6[L].astype(np.float64), -BITS * (L + 2)) for L in range(LEVELS - 2, -1, -1)),
                    ew + ev + 2)
    rel6 = np.linalg.norm(got6 - ref) / np.linalg.norm(ref)
    assert rel6 > 2 * rel


def test_item_key_bound():
    """m2l_i8_fkeys: keys per work item such that a level accumulator cannot overflow."""
    for m, want in ((4, 85), (5, 48), (6, 31)):
        n = (m + 1) ** 3
        nkq = (n + 15) // 16 * 16
        per_key = KS * 2 * nkq * 128 * 128
        assert (2 ** 31 - 1) // per_key == want
