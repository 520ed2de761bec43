"""ctypes front end of the C oracle tier (oracle/c/tlookup_oracle.c).  TEST INFRASTRUCTURE ONLY.

Arrays cross the boundary as numpy uint64 arrays of shape (n, 4): canonical Fr, little-endian
64-bit limbs.  `prove()` returns the same quantities as `oracle.tlookup.prove`.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "tlookup_oracle.c")
LIB = os.path.join(HERE, "c", "liboracle.so")
R = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001

ERRORS = {2: "E_SHAPE", 3: "E_NONCANONICAL", 4: "E_DUP_TABLE", 5: "E_NOT_IN_TABLE",
          6: "E_DIV_ZERO_T", 7: "E_DIV_ZERO_S", 8: "E_OOM"}


class OracleError(Exception):
    def __init__(self, code: int, index: int):
        super().__init__(f"{ERRORS.get(code, code)}({index})")
        self.code, self.name, self.index = code, ERRORS.get(code, str(code)), index


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wall", "-o", LIB, SRC])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        _lib.zko_tlookup.argtypes = [ctypes.c_uint64, ctypes.c_uint64, P, P, P, ctypes.c_int, ctypes.c_int,
                                     P, P, P, P, P, P, P, P, P]
        _lib.zko_tlookup.restype = ctypes.c_int
        _lib.zko_pair_inputs.argtypes = [ctypes.c_uint64, P, P, P, P]
        _lib.zko_tlookup_pair_stream.argtypes = [ctypes.c_uint64, ctypes.c_uint64, P, P, P, P, P, P, ctypes.c_int,
                                                 ctypes.c_int, P, P, P, P, P]
        _lib.zko_tlookup_pair_stream.restype = ctypes.c_int
        _lib.zko_int_inputs.argtypes = [ctypes.c_uint64, P, P]
        for f in ("zko_fr_mul", "zko_fr_add", "zko_fr_sub"):
            getattr(_lib, f).argtypes = [P, P, P]
        _lib.zko_fr_inv.argtypes = [P, P]
        _lib.zko_num_threads.restype = ctypes.c_int
        _lib.zko_set_threads.argtypes = [ctypes.c_int]
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def ints_to_limbs(xs: List[int]) -> np.ndarray:
    out = np.zeros((len(xs), 4), dtype=np.uint64)
    for i, x in enumerate(xs):
        for k in range(4):
            out[i, k] = (x >> (64 * k)) & 0xFFFFFFFFFFFFFFFF
    return out


def limbs_to_ints(a: np.ndarray) -> List[int]:
    a = np.asarray(a, dtype=np.uint64).reshape(-1, 4)
    return [int(r[0]) | (int(r[1]) << 64) | (int(r[2]) << 128) | (int(r[3]) << 192) for r in a]


def fr_binop(name: str, a: int, b: int) -> int:
    x, y, o = ints_to_limbs([a]), ints_to_limbs([b]), np.zeros((1, 4), np.uint64)
    getattr(lib(), f"zko_fr_{name}")(_p(x), _p(y), _p(o))
    return limbs_to_ints(o)[0]


def fr_inv(a: int) -> int:
    x, o = ints_to_limbs([a]), np.zeros((1, 4), np.uint64)
    lib().zko_fr_inv(_p(x), _p(o))
    return limbs_to_ints(o)[0]


def set_threads(n: int) -> None:
    lib().zko_set_threads(n)


def num_threads() -> int:
    return lib().zko_num_threads()


def inputs_from_workload(wl):
    """S, T as (n, 4) uint64 canonical limb arrays, built by the C oracle itself."""
    L = lib()
    S = np.zeros((wl.D, 4), dtype=np.uint64)
    T = np.zeros((wl.N, 4), dtype=np.uint64)
    if wl.kind == "int":
        s = np.ascontiguousarray(wl.s, dtype=np.int64)
        t = np.ascontiguousarray(wl.t, dtype=np.int64)
        L.zko_int_inputs(wl.D, _p(s), _p(S))
        L.zko_int_inputs(wl.N, _p(t), _p(T))
    else:
        af = ints_to_limbs([wl.chal.alpha_f % R])
        x = np.ascontiguousarray(wl.x, dtype=np.int32)
        y = np.ascontiguousarray(wl.y, dtype=np.int32)
        tx = np.ascontiguousarray(wl.tx, dtype=np.int32)
        ty = np.ascontiguousarray(wl.ty, dtype=np.int32)
        L.zko_pair_inputs(wl.D, _p(x), _p(y), _p(af), _p(S))
        L.zko_pair_inputs(wl.N, _p(tx), _p(ty), _p(af), _p(T))
    return S, T


def chal_array(beta, alpha1, alpha2, u, r) -> np.ndarray:
    return ints_to_limbs([beta % R, alpha1 % R, alpha2 % R] + [x % R for x in u] + [x % R for x in r])


class Result:
    def __init__(self, m, A, B, evals, finals):
        self.m, self.A, self.B, self.evals_limbs, self.finals_limbs = m, A, B, evals, finals

    @property
    def evals(self) -> List[List[int]]:
        v = limbs_to_ints(self.evals_limbs)
        return [v[4 * k:4 * k + 4] for k in range(len(v) // 4)]

    @property
    def finals(self):
        v = limbs_to_ints(self.finals_limbs)
        return dict(zip(["A", "S", "B", "T", "m"], v))


def prove(S: np.ndarray, T: np.ndarray, chal: np.ndarray, variant: int = 0, want_A: bool = True,
          want_B: bool = True) -> Result:
    D, N = S.shape[0], T.shape[0]
    d = D.bit_length() - 1
    m = np.zeros(N, dtype=np.uint32)
    A = np.zeros((D, 4), dtype=np.uint64) if want_A else None
    B = np.zeros((N, 4), dtype=np.uint64) if want_B else None
    ev = np.zeros((max(d, 1) * 4, 4), dtype=np.uint64)
    fin = np.zeros((5, 4), dtype=np.uint64)
    err = ctypes.c_int64(-1)
    S = np.ascontiguousarray(S, dtype=np.uint64)
    T = np.ascontiguousarray(T, dtype=np.uint64)
    st = lib().zko_tlookup(D, N, _p(S), _p(T), _p(chal), variant, 0, None, None, None,
                           _p(m), _p(A), _p(B), _p(ev), _p(fin), ctypes.byref(err))
    if st:
        raise OracleError(st, err.value)
    return Result(m, A, B, ev[:d * 4], fin)


def sumcheck(A: np.ndarray, S: np.ndarray, B: np.ndarray, T: np.ndarray, m: np.ndarray, chal: np.ndarray,
             variant: int = 0) -> Result:
    D, N = S.shape[0], T.shape[0]
    d = D.bit_length() - 1
    ev = np.zeros((max(d, 1) * 4, 4), dtype=np.uint64)
    fin = np.zeros((5, 4), dtype=np.uint64)
    err = ctypes.c_int64(-1)
    m = np.ascontiguousarray(m, dtype=np.uint32)
    args = [np.ascontiguousarray(x, dtype=np.uint64) for x in (S, T, A, B)]
    st = lib().zko_tlookup(D, N, _p(args[0]), _p(args[1]), _p(chal), variant, 1, _p(args[2]), _p(args[3]),
                           _p(m), None, None, None, _p(ev), _p(fin), ctypes.byref(err))
    if st:
        raise OracleError(st, err.value)
    return Result(m, None, None, ev[:d * 4], fin)


def prove_pair_stream(x, y, tx, ty, alpha_f: int, chal: np.ndarray, variant: int = 0, s: int = 4,
                      want_B: bool = True) -> Result:
    """The streaming tier (zko_tlookup_pair_stream): S_i = x_i + alpha_f y_i, T_j = tx_j + alpha_f ty_j (int32),
    first s rounds evaluated per aligned block of 2^s elements, memory ~ (D / 2^s) * 192 B + 8 B per lookup."""
    x = np.ascontiguousarray(x, dtype=np.int32)
    y = np.ascontiguousarray(y, dtype=np.int32)
    tx = np.ascontiguousarray(tx, dtype=np.int32)
    ty = np.ascontiguousarray(ty, dtype=np.int32)
    D, N = x.shape[0], tx.shape[0]
    d = D.bit_length() - 1
    af = ints_to_limbs([alpha_f % R])
    m = np.zeros(N, dtype=np.uint32)
    B = np.zeros((N, 4), dtype=np.uint64) if want_B else None
    ev = np.zeros((max(d, 1) * 4, 4), dtype=np.uint64)
    fin = np.zeros((5, 4), dtype=np.uint64)
    err = ctypes.c_int64(-1)
    st = lib().zko_tlookup_pair_stream(D, N, _p(x), _p(y), _p(tx), _p(ty), _p(af), _p(chal), variant, s, _p(m),
                                       _p(B), _p(ev), _p(fin), ctypes.byref(err))
    if st:
        raise OracleError(st, err.value)
    return Result(m, None, B, ev[:d * 4], fin)
