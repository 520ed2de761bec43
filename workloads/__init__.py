"""Seeded synthetic workloads shared by the oracle and the CUDA path.

This module is the ONE place both sides of the parity tests draw from.  It holds
no arithmetic of the tlookup method: it produces plain integer arrays (the
quantized tensors X, Y and the table columns T_X, T_Y) and uniformly random
challenges in [0, r).  Each side turns these into field elements itself:
the oracle with Python integers (oracle/), the GPU path with
`zkl_vec_import_i64` / `zkl_vec_import_pair` (a1 of SURVEY.md §8(a)).

Recipe (SURVEY.md §8(d) "Synthetic inputs"):

* splitmix64 counter generator: out(seed, i) = mix(seed + (i+1)*0x9E3779B97F4A7C15).
* challenges: chal(cfg, name, i) = SHA-256("zkl-v1/cfg{cfg}/{name}/{i}") as a
  little-endian integer, reduced mod r.  alpha2 = alpha1^2 (paper weights
  (1, alpha, alpha^2), Eq. tlookup-sumcheck-preliminary).
* C1 (range check): S_i = out(1, i) mod 256, T = [0, 256).
* C2/C3/H/C5 (activation function lookups): X ~ clamp(round(N(0, 4096^2))),
  T_X = [-32768, 32768), T_Y = round(4096 * f(x / 4096)); f = GELU (C2) or SiLU
  (C3, H, C5); S = X + alpha_f * Y, T = T_X + alpha_f * T_Y.  C3 zero-pads
  2048 x 11008 = 22,544,384 real entries to 2^25 ("zero-padding").
* C4 (zkAttn segment lookups, K=5, L=3, b=2^16):
  digits of the causal softmax gap; see `zkattn_digits`.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

# BLS12-381 scalar field modulus.  Only used to draw
# uniform challenges in [0, r) and to range-check inputs, never to compute.
R_MODULUS = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

CONFIG_SEEDS = {"1": 1, "2": 2, "3": 3, "5": 5, "H": 6}


def splitmix64(seed: int, idx: np.ndarray) -> np.ndarray:
    """out(seed, i) for an array of counters i (uint64, wrapping arithmetic)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def splitmix64_scalar(seed: int, i: int) -> int:
    m = (1 << 64) - 1
    z = (seed + (i + 1) * 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def chal(cfg: str, name: str, i: int) -> int:
    h = hashlib.sha256(f"zkl-v1/cfg{cfg}/{name}/{i}".encode("ascii")).digest()
    return int.from_bytes(h, "little") % R_MODULUS


@dataclass
class Challenges:
    beta: int
    alpha1: int
    alpha2: int
    u: List[int]          # u[0] pairs with the MSB coordinate (coordinate 0)
    r: List[int]          # r[k-1] is the challenge of round k (round 1 binds the LSB)
    alpha_f: int = 0      # function-lookup combiner, separate from alpha1


def challenges(cfg: str, d: int) -> Challenges:
    a1 = chal(cfg, "alpha1", 0)
    return Challenges(
        beta=chal(cfg, "beta", 0),
        alpha1=a1,
        alpha2=pow(a1, 2, R_MODULUS),
        u=[chal(cfg, "u", i) for i in range(d)],
        r=[chal(cfg, "r", i) for i in range(d)],
        alpha_f=chal(cfg, "alpha_f", 0),
    )


@dataclass
class Workload:
    """One tlookup instance as integer arrays.

    kind == "int":  S_i = s[i] (signed integer, x < 0 maps to r - |x|), T_j = t[j].
    kind == "pair": S_i = x[i] + alpha_f * y[i], T_j = tx[j] + alpha_f * ty[j].
    """
    name: str
    D: int
    N: int
    kind: str
    chal: Challenges
    s: Optional[np.ndarray] = None
    t: Optional[np.ndarray] = None
    x: Optional[np.ndarray] = None
    y: Optional[np.ndarray] = None
    tx: Optional[np.ndarray] = None
    ty: Optional[np.ndarray] = None
    meta: dict = field(default_factory=dict)

    @property
    def d(self) -> int:
        return self.D.bit_length() - 1

    @property
    def n(self) -> int:
        return self.N.bit_length() - 1


def _uniform01(seed: int, idx: np.ndarray) -> np.ndarray:
    return (splitmix64(seed, idx) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def gaussian(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Box-Muller standard normals from counters 2i, 2i+1 (float64)."""
    i = np.arange(start, start + count, dtype=np.uint64)
    u1 = _uniform01(seed, 2 * i)
    u2 = _uniform01(seed, 2 * i + 1)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


def _gelu(x: np.ndarray) -> np.ndarray:
    from scipy.special import erf
    return 0.5 * x * (1.0 + erf(x / math.sqrt(2.0)))


def _silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def activation_table(fn: str):
    tx = np.arange(-32768, 32768, dtype=np.int64)
    f = _gelu if fn == "gelu" else _silu
    ty = np.rint(4096.0 * f(tx / 4096.0)).astype(np.int64)
    return tx, ty


def range_check(D: int = 1 << 10, N: int = 1 << 8, cfg: str = "1", seed: int = 1) -> Workload:
    """C1: S_i = out(seed, i) mod N into T = [0, N)."""
    s = (splitmix64(seed, np.arange(D, dtype=np.uint64)) % np.uint64(N)).astype(np.int64)
    t = np.arange(N, dtype=np.int64)
    return Workload(f"C{cfg}-range", D, N, "int", challenges(cfg, D.bit_length() - 1), s=s, t=t)


def activation_x(cfg: str, start: int, count: int, real: int) -> np.ndarray:
    """X[start:start+count] of an activation workload (counter-based: any chunk can be drawn alone)."""
    x = np.rint(4096.0 * gaussian(CONFIG_SEEDS[cfg], count, start=start))
    x = np.clip(x, -32768, 32767).astype(np.int32)
    if real < start + count:
        x[max(0, real - start):] = 0
    return x


def activation(cfg: str = "H", D: Optional[int] = None, real: Optional[int] = None) -> Workload:
    """C2 (GELU, 2^20), C3 (SiLU, 22,544,384 -> 2^25), H (SiLU, 2^26), C5 (SiLU, 2^30)."""
    default_D = {"2": 1 << 20, "3": 1 << 25, "H": 1 << 26, "5": 1 << 30}[cfg]
    D = default_D if D is None else D
    if real is None:
        real = 2048 * 11008 if (cfg == "3" and D == default_D) else D
    fn = "gelu" if cfg == "2" else "silu"
    tx, ty = activation_table(fn)
    seed = CONFIG_SEEDS[cfg]
    x = np.rint(4096.0 * gaussian(seed, D))
    x = np.clip(x, -32768, 32767).astype(np.int32)
    if real < D:
        x[real:] = 0
    y = ty[x.astype(np.int64) + 32768].astype(np.int32)
    return Workload(f"C{cfg}-{fn}" if cfg != "H" else f"H-{fn}", D, 1 << 16, "pair",
                    challenges(cfg, D.bit_length() - 1),
                    x=x, y=y, tx=tx.astype(np.int32), ty=ty.astype(np.int32),
                    meta={"real": real, "fn": fn})


def zkattn_digits(k: int, heads: int = 32, seq: int = 2048) -> Workload:
    """C4 instance k (0..4): digit k of the causal softmax gap, K=5 segments of b=2^16.

    Flat index i = (h*seq + q)*seq + j.  Logits z ~ 3*N(0,1) for j <= q (counter
    stream 40); zhat_q = logsumexp_{j<=q} z; gap g = zhat_q - z >= 0.  Digit 4 =
    min(floor(g), 65535), digit 3 = floor(frac(g) * 65536), digits 0..2 uniform
    16-bit (stream 41).  Masked entries (j > q) saturate every digit to 0xffff.
    Instances 0-2 are range lookups into [0, 2^16); instances 3, 4 are function
    lookups x + alpha_f * T_Y^(k)[x] with T_Y^(3) = round(256 e^{-x/65536}) and
    T_Y^(4) = round(256 e^{-x}) (segment tables of).
    """
    D = heads * seq * seq
    qi = np.arange(seq)
    digits = np.empty(D, dtype=np.int64)
    for h in range(heads):
        base = h * seq * seq
        idx = np.arange(base, base + seq * seq, dtype=np.uint64)
        mask = (qi[None, :] > qi[:, None])          # j > q
        if k <= 2:
            v = ((splitmix64(41, idx) >> np.uint64(16 * k)) & np.uint64(0xFFFF)).astype(np.int64)
            v = v.reshape(seq, seq)
        else:
            z = 3.0 * gaussian(40, seq * seq, start=base).reshape(seq, seq)
            z = np.where(mask, -np.inf, z)
            zmax = np.max(z, axis=1, keepdims=True)
            zhat = zmax + np.log(np.sum(np.exp(z - zmax), axis=1, keepdims=True))
            g = np.where(mask, 0.0, zhat - z)
            if k == 4:
                v = np.minimum(np.floor(g), 65535).astype(np.int64)
            else:
                v = np.floor((g - np.floor(g)) * 65536.0).astype(np.int64)
        v = np.where(mask, 0xFFFF, v)
        digits[base:base + seq * seq] = v.reshape(-1)
    cfg = f"4.{k}"
    ch = challenges(cfg, D.bit_length() - 1)
    t = np.arange(1 << 16, dtype=np.int64)
    if k <= 2:
        return Workload(f"C4.{k}-digit", D, 1 << 16, "int", ch, s=digits, t=t)
    scale = 65536.0 if k == 3 else 1.0
    ty = np.rint(256.0 * np.exp(-t / scale)).astype(np.int64)
    return Workload(f"C4.{k}-segment", D, 1 << 16, "pair", ch,
                    x=digits.astype(np.int32), y=ty[digits].astype(np.int32),
                    tx=t.astype(np.int32), ty=ty.astype(np.int32))


def random_instance(D: int, N: int, seed: int, cfg: Optional[str] = None) -> Workload:
    """Small random instance: table = N distinct random 64-bit values, S drawn from it."""
    cfg = cfg or f"rand{seed}"
    idx = np.arange(N, dtype=np.uint64)
    t = (splitmix64(1000 + seed, idx) >> np.uint64(2)).astype(np.int64)
    # distinct by construction with overwhelming probability; enforce
    assert len(np.unique(t)) == N
    pick = (splitmix64(2000 + seed, np.arange(D, dtype=np.uint64)) % np.uint64(N)).astype(np.int64)
    return Workload(f"rand-{D}-{N}-{seed}", D, N, "int", challenges(cfg, D.bit_length() - 1),
                    s=t[pick], t=t)


def field_ints(w: Workload):
    """The canonical integers of S and T *as plain integers before reduction*.

    For kind "int" returns (s, t) as Python-int lists (negative values kept
    negative: each side maps x < 0 to r - |x| itself).  For "pair" returns None.
    """
    if w.kind != "int":
        return None
    return [int(v) for v in w.s], [int(v) for v in w.t]
