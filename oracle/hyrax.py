"""Hyrax / Pedersen commitments over BLS12-381 G1 — TEST INFRASTRUCTURE ONLY.

PAPER.md:187-203 (§3.4): Commit(S, r; pp) and ProveEval(S, [S], v, r; pp), instantiated by Hyrax, "a variant of the
Pedersen commitment that does not require a trusted setup", on a cyclic group with hard discrete log, homomorphic:
Commit(S1, r1) + Commit(S2, r2) = Commit(S1 + S2, r1 + r2); commitment size O(sqrt D).  Protocol 1 commits S, m
 and A, B; tlookup-Setup commits T with no hiding.

Readings:
* the group is BLS12-381 G1 (the curve of the scalar field): y^2 = x^3 + 4 over F_q;
* Hyrax layout: S (D = rows x cols, row-major) is a matrix; the commitment is one Pedersen vector commitment per row,
  C_j = sum_i S[j cols + i] G_i + rho_j H, with public generators G_0..G_{cols-1}, H ("no trusted setup": each is
  derived from a public label by hashing to the curve);
* hash to the curve by try-and-increment: x = LE-int(SHA256(tag || le32(i) || le32(ctr) || 0x00) ||
  SHA256(... || 0x01)) mod q, the first ctr with x^3 + 4 a square; y = (x^3 + 4)^((q+1)/4) (q = 3 mod 4), the
  smaller of y, q - y; then the cofactor h = #E / r is cleared (G = h P);
* ProveEval without the log-size inner-product argument: for v = (v_rows, v_cols) the prover sends
  w = sum_j e~(v_rows, j) S_row_j (a cols-vector) and y = <w, e~(v_cols, .)>; the verifier checks
  Com(w, sum_j e~ rho_j) = sum_j e~(v_rows, j) C_j and y.  (The O(log D) argument on w is out of scope.)
"""
import hashlib
from typing import List, Optional, Sequence, Tuple

from .field import R
from .mle import eq_table

# BLS12-381: z = -0xd201000000010000, r = z^4 - z^2 + 1, q = (z - 1)^2 r / 3 + z (pinned in the tests)
Q = 0x1A0111EA397FE69A4B1BA7B6434BACD764774B84F38512BF6730D2A0F6B0F6241EABFFFEB153FFFFB9FEFFFFFFFFAAAB
B_COEF = 4
H_COFACTOR = 0x396C8C005555E1568C00AAAB0000AAAB
G1_GEN = (0x17F1D3A73197D7942695638C4FA9AC0FC3688C4F9774B905A14E3A3F171BAC586C55E83FF97A1AEFFB3AF00ADB22C6BB,
          0x08B3F481E3AAA0F1A09E30ED741D8AE4FCF5E095D5D00AF600DB18CB2C04B3EDD03CC744A2888AE40CAA232946C5E7E1)

Point = Optional[Tuple[int, int]]   # affine (x, y), None = the point at infinity


def on_curve(P: Point) -> bool:
    if P is None:
        return True
    x, y = P
    return (y * y - x * x * x - B_COEF) % Q == 0


def neg(P: Point) -> Point:
    return None if P is None else (P[0], (-P[1]) % Q)


def add(P: Point, Qp: Point) -> Point:
    """Affine chord-and-tangent addition on y^2 = x^3 + 4 (a = 0)."""
    if P is None:
        return Qp
    if Qp is None:
        return P
    x1, y1 = P
    x2, y2 = Qp
    if x1 == x2:
        if (y1 + y2) % Q == 0:
            return None
        lam = 3 * x1 * x1 * pow(2 * y1, -1, Q) % Q
    else:
        lam = (y2 - y1) * pow(x2 - x1, -1, Q) % Q
    x3 = (lam * lam - x1 - x2) % Q
    return (x3, (lam * (x1 - x3) - y1) % Q)


def mul(k: int, P: Point) -> Point:
    """k P by double-and-add (the definition), k >= 0."""
    assert k >= 0
    acc, base = None, P
    while k:
        if k & 1:
            acc = add(acc, base)
        base = add(base, base)
        k >>= 1
    return acc


def hash_to_curve(tag: bytes, i: int) -> Point:
    """Try-and-increment into the order-r subgroup (reading above)."""
    ctr = 0
    while True:
        pre = tag + i.to_bytes(4, "little") + ctr.to_bytes(4, "little")
        x = int.from_bytes(hashlib.sha256(pre + b"\x00").digest() + hashlib.sha256(pre + b"\x01").digest(),
                           "little") % Q
        rhs = (x * x * x + B_COEF) % Q
        if rhs != 0 and pow(rhs, (Q - 1) // 2, Q) == 1:
            y = pow(rhs, (Q + 1) // 4, Q)
            y = min(y, Q - y)
            Pt = mul(H_COFACTOR, (x, y))
            if Pt is not None:
                return Pt
        ctr += 1


def generators(cols: int) -> Tuple[List[Point], Point]:
    """Public parameters: G_0..G_{cols-1} (tag "zkl-hyrax-G") and H (tag "zkl-hyrax-H", index 0)."""
    return [hash_to_curve(b"zkl-hyrax-G", i) for i in range(cols)], hash_to_curve(b"zkl-hyrax-H", 0)


def msm(scalars: Sequence[int], points: Sequence[Point]) -> Point:
    acc = None
    for s, P in zip(scalars, points):
        acc = add(acc, mul(s % R, P))
    return acc


def commit(S: Sequence[int], cols: int, G: Sequence[Point], Hb: Point, rho: Optional[Sequence[int]] = None):
    """Hyrax row commitments C_j = sum_i S[j cols + i] G_i + rho_j H (rho = None: no hiding)."""
    assert len(S) % cols == 0 and len(G) >= cols
    rows = len(S) // cols
    out = []
    for j in range(rows):
        C = msm(S[j * cols:(j + 1) * cols], G[:cols])
        if rho is not None:
            C = add(C, mul(rho[j] % R, Hb))
        out.append(C)
    return out


def prove_eval(S: Sequence[int], cols: int, v_rows: Sequence[int], v_cols: Sequence[int]):
    """w_i = sum_j e~(v_rows, j) S[j][i], y = sum_i w_i e~(v_cols, i) = S~(v_rows, v_cols) (rows = high bits)."""
    rows = len(S) // cols
    Er, Ec = eq_table(v_rows), eq_table(v_cols)
    assert len(Er) == rows and len(Ec) == cols
    w = [sum(Er[j] * S[j * cols + i] for j in range(rows)) % R for i in range(cols)]
    y = sum(a * b for a, b in zip(w, Ec)) % R
    return w, y


def verify_eval(C: Sequence[Point], cols: int, G: Sequence[Point], Hb: Point, v_rows, v_cols, w, y,
                rho: Optional[Sequence[int]] = None) -> bool:
    """sum_j e~(v_rows, j) C_j = Com(w, sum_j e~(v_rows, j) rho_j) and y = <w, e~(v_cols, .)>."""
    Er, Ec = eq_table(v_rows), eq_table(v_cols)
    lhs = msm(Er, C)
    rhs = msm(w, G[:cols])
    if rho is not None:
        rhs = add(rhs, mul(sum(e * p for e, p in zip(Er, rho)) % R, Hb))
    return lhs == rhs and y == sum(a * b for a, b in zip(w, Ec)) % R
