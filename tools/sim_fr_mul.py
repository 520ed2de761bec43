"""Word-level simulation of the aligned-pair CIOS schedule used by csrc/fr.cuh (dev check).

The q r1 product of each reduction step is not multiplied: r1 = 2^32 - 1, so q r1 = (q - 1) 2^32 + (2^32 - q) with
q = -x0, i.e. lo = x0 and hi = ~x0 + [x0 == 0] (three ALU instructions instead of an IMAD.HI pair).

Models every PTX carry chain with explicit 32-bit words and a carry flag, asserting that
the chains whose carry-out is dropped (Y chains) never produce a carry, for random and
extreme operands.  Not part of the oracle; a design check of the schedule only.
"""
import random
import sys

R = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
M = (1 << 32) - 1
rl = [(R >> (32 * i)) & M for i in range(8)]


class Chain:
    def __init__(self):
        self.c = 0

    def madc(self, a, b, add, hi, cc_in=True, cc_out=True):
        p = a * b
        v = ((p >> 32) if hi else (p & M)) + add + (self.c if cc_in else 0)
        self.c = (v >> 32) if cc_out else 0
        if not cc_out:
            assert v >> 32 == 0, "dropped carry"
        return v & M

    def add(self, a, b, cc_in=True, cc_out=True):
        v = a + b + (self.c if cc_in else 0)
        if not cc_out:
            assert v >> 32 == 0, "dropped carry"
        self.c = v >> 32
        return v & M


def mul(aw, bw):
    a = aw
    x = [0] * 9
    y = [0] * 8
    for i in range(8):
        b = bw[i]
        if i == 0:
            X = [0] * 9
            Y = [0] * 8
            for j in range(0, 8, 2):
                X[j] = (a[j] * b) & M
                X[j + 1] = (a[j] * b) >> 32
            for j in range(1, 8, 2):
                Y[j - 1] = (a[j] * b) & M
                Y[j] = (a[j] * b) >> 32
            X[8] = 0
        else:
            ch = Chain()
            X = [0] * 9
            Y = [0] * 8
            X[0] = ch.add(y[0], x[1], cc_in=False)
            src = x[2:9] + [0]
            for j in range(1, 8, 2):
                Y[j - 1] = ch.madc(a[j], b, src[j - 1], False)
                Y[j] = ch.madc(a[j], b, src[j], True, cc_out=(j != 7))
            ch = Chain()
            Xin = [X[0]] + y[1:8]
            for j in range(0, 8, 2):
                X[j] = ch.madc(a[j], b, Xin[j], False, cc_in=(j != 0))
                X[j + 1] = ch.madc(a[j], b, Xin[j + 1], True)
            X[8] = ch.add(0, 0, cc_out=False)
        q = (-X[0]) & M
        xo = X[0]
        hi1 = ((~xo) + (1 if xo == 0 else 0)) & M   # hi(q r1) for r1 = 2^32 - 1 (lo(q r1) = xo): no multiply
        assert (hi1 << 32) + xo == q * rl[1]
        ch = Chain()
        X[0] = ch.add(X[0], q, cc_in=False)
        assert X[0] == 0
        X[1] = ch.add(X[1], 0)
        for j in range(2, 8, 2):
            X[j] = ch.madc(q, rl[j], X[j], False)
            X[j + 1] = ch.madc(q, rl[j], X[j + 1], True)
        X[8] = ch.add(X[8], 0, cc_out=False)
        ch = Chain()
        Y[0] = ch.add(Y[0], xo, cc_in=False)
        Y[1] = ch.add(Y[1], hi1)
        for j in range(3, 8, 2):
            Y[j - 1] = ch.madc(q, rl[j], Y[j - 1], False)
            Y[j] = ch.madc(q, rl[j], Y[j], True, cc_out=(j != 7))
        x, y = X, Y
    ch = Chain()
    t = []
    for k in range(8):
        t.append(ch.add(x[k + 1], y[k], cc_in=(k != 0), cc_out=(k != 7)))
    v = sum(w << (32 * k) for k, w in enumerate(t))
    assert v < 2 * R
    return v - R if v >= R else v


def words(v):
    return [(v >> (32 * i)) & M for i in range(8)]


def main(n):
    rng = random.Random(1)
    Rinv = pow(1 << 256, -1, R)
    edge = [0, 1, R - 1, R - 2, (1 << 255) % R, R // 2, (1 << 224) - 1, M, R - M]
    vals = edge + [rng.randrange(R) for _ in range(n)]
    # adversarial: limbs all 0xffffffff where allowed
    vals += [R - 1 - (rng.randrange(1 << 32) << (32 * rng.randrange(8))) % R for _ in range(n // 4)]
    cnt = 0
    for i, a in enumerate(vals):
        for b in (vals[(i * 13 + 5) % len(vals)], a, R - 1):
            got = mul(words(a), words(b))
            assert got == a * b * Rinv % R, (hex(a), hex(b))
            cnt += 1
    print("ok", cnt)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 20000)
