"""The verifier's side of the Fiat-Shamir transcript, with hashlib.  Test infrastructure."""
import hashlib

R = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


def _chal(h: bytes, label: bytes, i: int) -> int:
    return int.from_bytes(hashlib.sha256(h + label + i.to_bytes(4, "little")).digest(), "little") % R


def derive(seed: bytes, D: int, N: int, variant: int, evals):
    """Replays the transcript: (beta, alpha1, alpha2, u, r) from the seed and the prover's round polynomials."""
    d = D.bit_length() - 1
    h = hashlib.sha256(b"zkl-fs-v1" + seed + D.to_bytes(8, "little") + N.to_bytes(8, "little")
                       + variant.to_bytes(4, "little")).digest()
    beta, a1 = _chal(h, b"beta", 0), _chal(h, b"alpha", 0)
    u = [_chal(h, b"u", c) for c in range(d)]
    r = []
    for k in range(1, d + 1):
        h = hashlib.sha256(h + b"g" + k.to_bytes(4, "little")
                           + b"".join(int(x).to_bytes(32, "little") for x in evals[k - 1])).digest()
        r.append(_chal(h, b"r", k))
    return {"beta": beta, "alpha1": a1, "alpha2": a1 * a1 % R, "u": u, "r": r}
