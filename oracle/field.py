"""Fr, the BLS12-381 scalar field, with Python integers (TEST INFRASTRUCTURE ONLY).

PAPER.md:543 (§6.2, "|F| ~ 2^254", BLS12-381) and PAPER.md:627 (§7, BLS12-381 via
ec-gpu / mcl).  The modulus value is SURVEY.md Appendix A (reading 1 of DESIGN.md).
Every element is a canonical integer in [0, r).
"""

R = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


class NotInvertible(ZeroDivisionError):
    pass


def fr(x: int) -> int:
    """Integer -> Fr.  Negative quantized values x < 0 map to r - |x| (reading 15)."""
    return x % R


def add(a: int, b: int) -> int:
    return (a + b) % R


def sub(a: int, b: int) -> int:
    return (a - b) % R


def neg(a: int) -> int:
    return (-a) % R


def mul(a: int, b: int) -> int:
    return (a * b) % R


def inv(a: int) -> int:
    """Textbook modular inverse (library routine: extended Euclid inside pow)."""
    if a % R == 0:
        raise NotInvertible("inverse of 0")
    return pow(a, -1, R)


def to_bytes(a: int) -> bytes:
    """Canonical 32-byte little-endian encoding."""
    assert 0 <= a < R
    return a.to_bytes(32, "little")


def from_bytes(b: bytes) -> int:
    return int.from_bytes(b, "little")
