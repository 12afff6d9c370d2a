"""Pins for oracle.fp16 (P1 of SURVEY.md §8c.4): IEEE binary16 closed forms + SPEC examples."""
import numpy as np

from conftest import golden_lines
from oracle.fp16 import fl16, pow2_colscale


def _parse(tok):
    return float.fromhex(tok) if tok.startswith(("0x", "-0x")) else float(tok)


def test_golden_fp16_examples():
    n = 0
    for line in golden_lines("fp16_rounding.txt"):
        x, bits = line.split()[:2]
        got = np.float16(fl16(np.array([_parse(x)]))[0]).view(np.uint16)
        assert int(got) == int(bits, 16), (x, hex(int(got)), bits)
        n += 1
    assert n >= 8


def test_fp16_closed_form_random():
    # For normal-range x: |fl16(x) - x| <= 2^-11 |x| and fl16(x) has at most 11 significant bits.
    rng = np.random.default_rng(0)
    x = rng.standard_normal(20000) * np.exp2(rng.integers(-13, 15, 20000))
    x = x[(np.abs(x) >= 2.0 ** -14) & (np.abs(x) <= 65504.0)]      # normal binary16 range
    y = fl16(x)
    assert np.all(np.abs(y - x) <= np.ldexp(np.abs(x), -11))
    m, e = np.frexp(y)
    assert np.all(np.ldexp(m, 11) == np.round(np.ldexp(m, 11)))
    # Rounding is to NEAREST: no other 11-bit neighbour is closer.
    ulp = np.ldexp(1.0, e - 11)
    assert np.all(np.abs(y - x) <= ulp / 2 + 0.0)


def test_pow2_colscale_range():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((50, 7)) * np.exp2(rng.integers(-40, 30, 7))
    x[:, 3] = 0.0
    s = pow2_colscale(x)
    mx = np.max(np.abs(x * s), axis=0)
    nz = np.arange(7) != 3
    assert np.all((mx[nz] >= 1.0) & (mx[nz] < 2.0))
    assert s[3] == 1.0
    _, e = np.frexp(s)
    assert np.all(np.frexp(s)[0] == 0.5)  # exact powers of two
    # exact boundary: max exactly a power of two maps to 1
    z = np.array([[0.25, -8.0], [0.125, 4.0]])
    assert np.array_equal(np.max(np.abs(z * pow2_colscale(z)), axis=0), [1.0, 1.0])
