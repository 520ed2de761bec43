"""Multilinear extensions and eq, as defined in PAPER.md §3.3 (TEST INFRASTRUCTURE ONLY).

PAPER.md:168  tensor <-> function on {0,1}^d, "writing indices in binary format".
PAPER.md:168-170 (Eq. MLE)  S~(u) = sum_i e~(u, i) S(i),
PAPER.md:170  e~(u, v) printed as a SUM over coordinates; read as the PRODUCT
              prod_c (u_c v_c + (1 - u_c)(1 - v_c)) — the only form that "reduces
              to the equality indicator" (reading 2).
Bit order: coordinate 0 is the most significant bit of the row-major flat index
(reading 3).
"""
from typing import List, Sequence

from .field import R


def bits_msb_first(i: int, d: int) -> List[int]:
    """Binary representation of index i in d bits, coordinate 0 = MSB."""
    return [(i >> (d - 1 - c)) & 1 for c in range(d)]


def eq(u: Sequence[int], v: Sequence[int]) -> int:
    """e~(u, v) = prod_c (u_c v_c + (1 - u_c)(1 - v_c))  (product reading)."""
    assert len(u) == len(v)
    acc = 1
    for uc, vc in zip(u, v):
        acc = acc * ((uc * vc + (1 - uc) * (1 - vc)) % R) % R
    return acc


def eq_table(u: Sequence[int]) -> List[int]:
    """[e~(u, bits(i)) for i in [0, 2^d)] — each entry by the definition."""
    d = len(u)
    return [eq(u, bits_msb_first(i, d)) for i in range(1 << d)]


def mle_eval(vals: Sequence[int], point: Sequence[int]) -> int:
    """S~(point) = sum_i e~(point, bits(i)) S_i   (Eq. MLE)."""
    d = len(point)
    assert len(vals) == 1 << d
    acc = 0
    for i, s in enumerate(vals):
        acc = (acc + eq(point, bits_msb_first(i, d)) * s) % R
    return acc
