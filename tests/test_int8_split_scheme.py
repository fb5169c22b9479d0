"""CPU checks of the arithmetic behind the int8-split FD path (the CUDA kernels are in
paper_1705_04384_b200/csrc/oz.cu, parity against the oracle in test_gpu_int8.py).  Written from the scheme's
definition, independently of the kernels:

  q = floor(x 2^(62 - e)) with max|x| < 2^e;  a_0 = q >> 55 (signed byte), a_i = (q >> (55 - 8 i)) & 255 (i = 1..6)
  x ~ 2^(e - 62) sum_i a_i 2^(55 - 8 i)
  sum_k f_k x_k ~ 2^(e_f + e_x - 124) sum_{t <= 7} 2^(110 - 8 t) C_t,  C_t = sum_{i + j = t} sum_k f_{k,j} x_{k,i}
"""
import numpy as np
import pytest

S, NW = 7, 8


def exponent(row):
    m = np.max(np.abs(row))
    return 0 if m == 0 else int(np.frexp(m)[1])


def digits(row, e):
    """Exact integer digits of a row (python ints: no overflow, no rounding)."""
    out = np.zeros((S, row.size), dtype=np.int64)
    for k, v in enumerate(row):
        q = int(np.floor(np.ldexp(v, 62 - e)))  # exact: a power-of-two scaling, then floor
        assert -(1 << 62) <= q < (1 << 62)
        out[0, k] = q >> 55  # arithmetic shift: signed
        for i in range(1, S):
            out[i, k] = (q >> (55 - 8 * i)) & 255
    return out


def reconstruct(d, e):
    return sum(np.ldexp(d[i].astype(np.float64), e - 62 + 55 - 8 * i) for i in range(S))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_digit_ranges_and_reconstruction(seed):
    rng = np.random.default_rng(seed)
    row = rng.standard_normal(256) * np.exp(rng.uniform(-20, 20, 256))
    e = exponent(row)
    d = digits(row, e)
    assert d[0].min() >= -128 and d[0].max() <= 127           # signed leading byte
    assert d[1:].min() >= 0 and d[1:].max() <= 255            # unsigned lower bytes
    # truncated below bit 7 of q: the error is below 2^(e - 55) for every element
    assert np.max(np.abs(reconstruct(d, e) - row)) <= np.ldexp(1.0, e - 55)


def pair_sums(dx, df):
    """C_t for the kept weights t = i + j < NW (exact python ints)."""
    C = [0] * NW
    for i in range(S):
        for j in range(S):
            if i + j < NW:
                C[i + j] += int(np.dot(dx[i].astype(object), df[j].astype(object)))
    return C


@pytest.mark.parametrize("K,seed", [(1, 0), (131, 1), (256, 2), (512, 3)])
def test_int32_accumulators_do_not_overflow(K, seed):
    # worst case: every digit at its extreme (|a_0| = 128, a_i = 255), 7 pairs in one weight
    worst = max(128 * 255, 255 * 255) * K * 7
    assert worst < 2 ** 31, (K, worst)
    rng = np.random.default_rng(seed)
    x, f = rng.standard_normal(K), rng.standard_normal(K)
    C = pair_sums(digits(x, exponent(x)), digits(f, exponent(f)))
    assert max(abs(c) for c in C) < 2 ** 31


@pytest.mark.parametrize("K,seed,scale", [(64, 0, 0.0), (131, 1, 30.0), (256, 2, 5.0), (512, 3, 0.0)])
def test_dot_product_matches_fp64_rounding_level(K, seed, scale):
    # the scheme's dot product against an exact (rational) reference: error at the level of the FP64 dot
    # product's own rounding, relative to sum |f_k x_k|, also for rows with a large dynamic range
    from fractions import Fraction
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(K) * np.exp(rng.uniform(-scale, scale, K))
    f = rng.standard_normal(K)
    ex, ef = exponent(x), exponent(f)
    C = pair_sums(digits(x, ex), digits(f, ef))
    acc = sum(C[t] * (1 << (8 * (NW - 1 - t))) for t in range(NW))  # exact integer
    y = np.ldexp(float(acc), ex + ef - 70)  # one rounding, as in the kernel's epilogue (up to the split sum)
    exact = float(sum(Fraction(a) * Fraction(b) for a, b in zip(x, f)))
    mag = float(np.sum(np.abs(x * f)))
    # FP64-like rounding of the result, plus the scheme's own truncation (2^-55 of each row scale per element)
    # and the dropped digit pairs (five u8 x u8 pairs at weight 2^-78): both relative to 2^(e_x + e_f)
    scheme = (2 * K * 2.0 ** -55 + 5 * 255 ** 2 * K * 2.0 ** -78) * np.ldexp(1.0, ex + ef)
    assert abs(y - exact) <= 4 * 2.0 ** -52 * mag + scheme


def test_zero_row_has_zero_digits():
    z = np.zeros(16)
    assert exponent(z) == 0
    assert not digits(z, 0).any()
