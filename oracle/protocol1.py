"""Protocol 1 (tlookup) with its commitments, non-interactive -- TEST INFRASTRUCTURE ONLY.

The function-lookup form of PAPER.md:287: the prover shows Y = f(X) elementwise by X + alpha Y in T_X + alpha T_Y.
Every message is bound into a SHA-256 transcript before the challenge that follows it (the order of Protocol 1):

  h = SHA256("zkl-p1-v1" || seed[32] || le64(D) || le64(N) || le32(variant) || le64(cols))
  absorb(label, C) : h = SHA256(h || label || le32(#C) || C_0 || C_1 ...), a point = x (48 B LE) || y (48 B LE) ||
                     1 byte (1 = the point at infinity, coordinates 0)
  chal(label, i)   = LE-int(SHA256(h || label || le32(i))) mod r
  [T_X] "TX", [T_Y] "TY"  (tlookup-Setup: Commit(T; 0)), [X] "X", [Y] "Y"   ->  alpha_f = chal("alpha_f", 0)
  S = X + alpha_f Y, T = T_X + alpha_f T_Y; [S] = [X] + alpha_f [Y] by homomorphism
  m (Eq. hab22-coefs), [m] "m"  (tlookup-Prep)                          ->  beta = chal("beta", 0)
  A, B (Eq. hab22-invs), [A] "A", [B] "B"        ->  alpha1 = chal("alpha", 0), u_c = chal("u", c)
  the sumcheck of Eq. tlookup-sumcheck: h_k = SHA256(h || "g" || le32(k) || g_k(0..3)), r_k = chal("r", k)
  proofs of evaluation on [A], [S] (through [X], [Y]), [B], [T] (through [T_X], [T_Y]) and [m] at
  v = (r_d, ..., r_1) and v' = v[d-n:] (row-restriction Hyrax, oracle/hyrax.py; no hiding in this build).

`prove` is the definition written out with the oracle's own pieces (multiplicities, inverses, sumcheck_prove, Hyrax
commit / prove_eval); `verify` checks a proof from its commitments and messages alone.
"""
import hashlib
from typing import Dict, List, Sequence

from . import hyrax as HX
from . import tlookup as TL
from .field import R

TAG = b"zkl-p1-v1"


def point_bytes(P) -> bytes:
    if P is None:
        return bytes(96) + b"\x01"
    return P[0].to_bytes(48, "little") + P[1].to_bytes(48, "little") + b"\x00"


def absorb(h: bytes, label: bytes, C: Sequence) -> bytes:
    return hashlib.sha256(h + label + len(C).to_bytes(4, "little") + b"".join(point_bytes(P) for P in C)).digest()


def chal(h: bytes, label: bytes, i: int) -> int:
    return int.from_bytes(hashlib.sha256(h + label + i.to_bytes(4, "little")).digest(), "little") % R


def h0(seed: bytes, D: int, N: int, variant: int, cols: int) -> bytes:
    return hashlib.sha256(TAG + seed + D.to_bytes(8, "little") + N.to_bytes(8, "little") +
                          variant.to_bytes(4, "little") + cols.to_bytes(8, "little")).digest()


def absorb_round(h: bytes, k: int, g: Sequence[int]) -> bytes:
    return hashlib.sha256(h + b"g" + k.to_bytes(4, "little") + b"".join(int(x).to_bytes(32, "little") for x in g)).digest()


def _points(D, cols, v):
    """v (length log2 D, coordinate 0 = MSB) -> (row part, column part) of the Hyrax layout (rows = high bits)."""
    lr = (D // cols).bit_length() - 1
    return v[:lr], v[lr:]


def prove(x: Sequence[int], y: Sequence[int], tx: Sequence[int], ty: Sequence[int], seed: bytes, cols: int,
          variant: int = TL.PAPER, G=None, H=None) -> Dict:
    D, N = len(x), len(tx)
    d, n = D.bit_length() - 1, N.bit_length() - 1
    if G is None:
        G, H = HX.generators(cols)
    X = [v % R for v in x]
    Y = [v % R for v in y]
    TX = [v % R for v in tx]
    TY = [v % R for v in ty]
    C = {"TX": HX.commit(TX, cols, G, H), "TY": HX.commit(TY, cols, G, H),
         "X": HX.commit(X, cols, G, H), "Y": HX.commit(Y, cols, G, H)}
    h = h0(seed, D, N, variant, cols)
    for lab in ("TX", "TY", "X", "Y"):
        h = absorb(h, lab.encode(), C[lab])
    af = chal(h, b"alpha_f", 0)
    S = [(a + af * b) % R for a, b in zip(X, Y)]
    T = [(a + af * b) % R for a, b in zip(TX, TY)]
    m = TL.multiplicities(S, T)
    C["m"] = HX.commit([c % R for c in m], cols, G, H)
    h = absorb(h, b"m", C["m"])
    beta = chal(h, b"beta", 0)
    A, B = TL.inverses(S, T, beta, m, variant)
    C["A"] = HX.commit(A, cols, G, H)
    C["B"] = HX.commit(B, cols, G, H)
    h = absorb(h, b"A", C["A"])
    h = absorb(h, b"B", C["B"])
    a1 = chal(h, b"alpha", 0)
    ch = TL.Challenges(beta, a1, a1 * a1 % R, [chal(h, b"u", c) for c in range(d)], [])
    state = {"h": h}

    def next_r(k, g):
        state["h"] = absorb_round(state["h"], k, g)
        return chal(state["h"], b"r", k)

    tr = TL.sumcheck_prove(A, S, B, T, m, ch, variant, next_r=next_r)
    v = [ch.r[d - c - 1] for c in range(d)]
    vt = v[d - n:]
    ev = {}
    for lab, vec, pt, L in (("A", A, v, D), ("X", X, v, D), ("Y", Y, v, D), ("TX", TX, vt, N), ("TY", TY, vt, N),
                            ("m", [c % R for c in m], vt, N), ("B", B, vt, N)):
        vr, vc = _points(L, cols, pt)
        ev[lab] = HX.prove_eval(vec, cols, vr, vc)
    return {"D": D, "N": N, "cols": cols, "variant": variant, "seed": seed, "C": C, "alpha_f": af,
            "challenges": ch, "evals": tr.evals, "finals": tr.finals, "eval_proofs": ev}


def verify(pf: Dict, G=None, H=None) -> bool:
    """Check a Protocol-1 proof from its messages: the transcript's challenges, the sumcheck (with g_d(r_d) = f(v)
    from the finals), and every final against its commitment through a proof of evaluation."""
    D, N, cols, variant = pf["D"], pf["N"], pf["cols"], pf["variant"]
    d, n = D.bit_length() - 1, N.bit_length() - 1
    if G is None:
        G, H = HX.generators(cols)
    C = pf["C"]
    h = h0(pf["seed"], D, N, variant, cols)
    for lab in ("TX", "TY", "X", "Y"):
        h = absorb(h, lab.encode(), C[lab])
    af = chal(h, b"alpha_f", 0)
    h = absorb(h, b"m", C["m"])
    beta = chal(h, b"beta", 0)
    h = absorb(h, b"A", C["A"])
    h = absorb(h, b"B", C["B"])
    a1 = chal(h, b"alpha", 0)
    u = [chal(h, b"u", c) for c in range(d)]
    r = []
    for k in range(1, d + 1):
        h = absorb_round(h, k, pf["evals"][k - 1])
        r.append(chal(h, b"r", k))
    ch = TL.Challenges(beta, a1, a1 * a1 % R, u, r)
    if af != pf["alpha_f"]:
        return False
    if not TL.verify(TL.Transcript(pf["evals"], pf["finals"]), D, N, ch, variant):
        return False
    v = [r[d - c - 1] for c in range(d)]
    vt = v[d - n:]
    ev = pf["eval_proofs"]
    for lab, pt, L in (("A", v, D), ("X", v, D), ("Y", v, D), ("TX", vt, N), ("TY", vt, N), ("m", vt, N),
                       ("B", vt, N)):
        vr, vc = _points(L, cols, pt)
        w, yv = ev[lab]
        if not HX.verify_eval(C[lab], cols, G, H, vr, vc, w, yv):
            return False
    f = pf["finals"]
    return (ev["A"][1] == f["A"] and (ev["X"][1] + af * ev["Y"][1]) % R == f["S"] and ev["B"][1] == f["B"]
            and (ev["TX"][1] + af * ev["TY"][1]) % R == f["T"] and ev["m"][1] == f["m"])
