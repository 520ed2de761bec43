"""Word-level simulation of the aligned-pair CIOS schedule of fq_mul in csrc/g1.cuh (dev check).

The F_q analogue of tools/sim_fr_mul.py: 12 x 32-bit limbs, R = 2^384, the generic reduction multiplier
m = x0 q' mod 2^32 (q' = -q^{-1} mod 2^32) and all twelve words of q multiplied.  The running value is
X + Y 2^32 with X (13 words) aligned at word 0 and Y (12 words) aligned at word 1, so every lo/hi product pair
lands on an aligned register pair (one IMAD.WIDE.U32 each).  Every PTX carry chain is modelled with explicit
32-bit words and a carry flag, asserting that the chains whose carry-out is dropped never produce one, for random
and extreme operands.  Not part of the oracle; a design check of the schedule only.
"""
import random
import sys

Q = 0x1A0111EA397FE69A4B1BA7B6434BACD764774B84F38512BF6730D2A0F6B0F6241EABFFFEB153FFFFB9FEFFFFFFFFAAAB
M = (1 << 32) - 1
ql = [(Q >> (32 * i)) & M for i in range(12)]
QP = (-pow(Q, -1, 1 << 32)) % (1 << 32)


class Chain:
    def __init__(self):
        self.c = 0

    def madc(self, a, b, add, hi, cc_in=True, cc_out=True):
        p = a * b
        v = ((p >> 32) if hi else (p & M)) + add + (self.c if cc_in else 0)
        if not cc_out:
            assert v >> 32 == 0, "dropped carry"
        self.c = v >> 32
        return v & M

    def add(self, a, b, cc_in=True, cc_out=True):
        v = a + b + (self.c if cc_in else 0)
        if not cc_out:
            assert v >> 32 == 0, "dropped carry"
        self.c = v >> 32
        return v & M


def reduce_step(X, Y):
    m = (X[0] * QP) & M
    ch = Chain()
    for j in range(0, 12, 2):
        X[j] = ch.madc(m, ql[j], X[j], False, cc_in=(j != 0))
        X[j + 1] = ch.madc(m, ql[j], X[j + 1], True)
    X[12] = ch.add(X[12], 0, cc_out=False)
    assert X[0] == 0
    ch = Chain()
    for j in range(1, 12, 2):
        Y[j - 1] = ch.madc(m, ql[j], Y[j - 1], False, cc_in=(j != 1))
        Y[j] = ch.madc(m, ql[j], Y[j], True, cc_out=(j != 11))


def mul(a, bw):
    X = [0] * 13
    Y = [0] * 12
    b = bw[0]
    for j in range(0, 12, 2):
        X[j], X[j + 1] = (a[j] * b) & M, (a[j] * b) >> 32
    for j in range(1, 12, 2):
        Y[j - 1], Y[j] = (a[j] * b) & M, (a[j] * b) >> 32
    reduce_step(X, Y)
    for i in range(1, 12):
        b = bw[i]
        x, y = X, Y
        X = [0] * 13
        Y = [0] * 12
        ch = Chain()
        M0 = ch.add(y[0], x[1], cc_in=False)
        src = x[2:13] + [0]
        for j in range(1, 12, 2):
            Y[j - 1] = ch.madc(a[j], b, src[j - 1], False)
            Y[j] = ch.madc(a[j], b, src[j], True, cc_out=(j != 11))
        ch = Chain()
        Xin = [M0] + y[1:12]
        for j in range(0, 12, 2):
            X[j] = ch.madc(a[j], b, Xin[j], False, cc_in=(j != 0))
            X[j + 1] = ch.madc(a[j], b, Xin[j + 1], True)
        X[12] = ch.add(0, 0, cc_out=False)
        reduce_step(X, Y)
    ch = Chain()
    t = [ch.add(X[k + 1], Y[k], cc_in=(k != 0), cc_out=(k != 11)) for k in range(12)]
    v = sum(w << (32 * k) for k, w in enumerate(t))
    assert v < 2 * Q
    return v - Q if v >= Q else v


def words(v):
    return [(v >> (32 * i)) & M for i in range(12)]


def main(n):
    rng = random.Random(1)
    Rinv = pow(1 << 384, -1, Q)
    edge = [0, 1, 2, Q - 1, Q - 2, Q // 2, (1 << 380) - 1, M, Q - M, (1 << 352) - 1, Q - (1 << 352)]
    vals = edge + [rng.randrange(Q) for _ in range(n)]
    vals += [Q - 1 - (rng.randrange(1 << 32) << (32 * rng.randrange(12))) % Q for _ in range(n // 4)]
    cnt = 0
    for i, a in enumerate(vals):
        for b in (vals[(i * 13 + 5) % len(vals)], a, Q - 1):
            got = mul(words(a), words(b))
            assert got == a * b * Rinv % Q, (hex(a), hex(b))
            cnt += 1
    print("ok", cnt)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 20000)
