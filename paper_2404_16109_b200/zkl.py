"""Thin Python binding of the zkl C ABI (include/zkl.h) — argument marshalling only.

Every step of the tlookup path runs in libzkl.so (hand-written sm_100a CUDA).  PyTorch provides the
device memory (field vectors, the workspace, table memory) and the CUDA stream.  There is no CPU
fallback: if libzkl.so is missing or no GPU is present, calls fail loudly.

C names are exposed unchanged (`zkl_tlookup_prepare`, ...); `Context` bundles the common calls.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZKL_LIB") or os.path.join(HERE, "libzkl.so")   # ZKL_LIB: experiment builds (tools only)
R_MODULUS = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001

STATUS = ["ZKL_OK", "ZKL_E_ARG", "ZKL_E_SHAPE", "ZKL_E_NONCANONICAL", "ZKL_E_DUP_TABLE", "ZKL_E_NOT_IN_TABLE",
          "ZKL_E_DIV_ZERO_T", "ZKL_E_DIV_ZERO_S", "ZKL_E_CUDA", "ZKL_E_NCCL", "ZKL_E_OOM", "ZKL_E_STATE"]
PAPER, LOGUP = 0, 1


class zkl_fr(ctypes.Structure):
    _fields_ = [("w", ctypes.c_uint32 * 8)]


class zkl_g1(ctypes.Structure):
    _fields_ = [("x", ctypes.c_uint32 * 12), ("y", ctypes.c_uint32 * 12), ("infinity", ctypes.c_uint32)]


def g1_to_py(p: "zkl_g1"):
    """Affine point -> (x, y) Python ints, or None for the point at infinity."""
    if p.infinity:
        return None
    return (sum(int(p.x[i]) << (32 * i) for i in range(12)), sum(int(p.y[i]) << (32 * i) for i in range(12)))


class zkl_vec(ctypes.Structure):
    _fields_ = [("limbs", ctypes.c_void_p), ("n", ctypes.c_uint64)]


class zkl_challenges(ctypes.Structure):
    _fields_ = [("beta", zkl_fr), ("alpha1", zkl_fr), ("alpha2", zkl_fr),
                ("u", ctypes.POINTER(zkl_fr)), ("r", ctypes.POINTER(zkl_fr))]


class zkl_final_evals(ctypes.Structure):
    _fields_ = [("A", zkl_fr), ("S", zkl_fr), ("B", zkl_fr), ("T", zkl_fr), ("m", zkl_fr)]


_G1P, _FRP = ctypes.POINTER(zkl_g1), ctypes.POINTER(zkl_fr)


class zkl_p1_proof(ctypes.Structure):
    _fields_ = [("C_X", _G1P), ("C_Y", _G1P), ("C_TX", _G1P), ("C_TY", _G1P), ("C_m", _G1P), ("C_A", _G1P),
                ("C_B", _G1P), ("round_evals", _FRP), ("finals", zkl_final_evals), ("alpha_f", zkl_fr),
                ("derived", _FRP), ("w_A", _FRP), ("w_X", _FRP), ("w_Y", _FRP), ("w_TX", _FRP), ("w_TY", _FRP),
                ("w_m", _FRP), ("w_B", _FRP), ("y_A", zkl_fr), ("y_X", zkl_fr), ("y_Y", zkl_fr), ("y_TX", zkl_fr),
                ("y_TY", zkl_fr), ("y_m", zkl_fr), ("y_B", zkl_fr)]


class ZklError(RuntimeError):
    def __init__(self, status: int, index: int = -1, msg: str = ""):
        name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{name}({index}): {msg}")
        self.status, self.name, self.index = status, name, index


_lib = None


def lib() -> ctypes.CDLL:
    """Load libzkl.so (built in-tree by paper_2404_16109_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2404_16109_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P, U64, I32, I64P = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)
        sig = {
            "zkl_strerror": ([I32], ctypes.c_char_p),
            "zkl_ctx_create": ([I32, P, ctypes.POINTER(P)], I32),
            "zkl_nccl_unique_id": ([ctypes.c_char_p], I32),
            "zkl_ctx_create_dist": ([I32, P, ctypes.c_char_p, I32, I32, ctypes.POINTER(P)], I32),
            "zkl_ctx_destroy": ([P], None),
            "zkl_group_create": ([I32, I32, U64, U64, ctypes.POINTER(P)], I32),
            "zkl_group_destroy": ([P], None),
            "zkl_ctx_create_loopback": ([I32, P, P, I32, ctypes.POINTER(P)], I32),
            "zkl_last_error": ([P], ctypes.c_char_p),
            "zkl_workspace_bytes": ([U64, U64, I32], ctypes.c_size_t),
            "zkl_ctx_set_workspace": ([P, P, ctypes.c_size_t], I32),
            "zkl_ctx_launch_count": ([P], U64),
            "zkl_ctx_set_profiling": ([P, I32], I32),
            "zkl_ctx_set_async": ([P, I32], I32),
            "zkl_matmul_workspace_bytes": ([U64, U64, U64], ctypes.c_size_t),
            "zkl_hyrax_pp_bytes": ([U64], ctypes.c_size_t),
            "zkl_table_attach_pair": ([P, P, P, P, ctypes.POINTER(zkl_fr)], I32),
            "zkl_hyrax_setup": ([P, U64, P, ctypes.c_size_t], I32),
            "zkl_hyrax_export_generators": ([P, P, U64, P], I32),
            "zkl_hyrax_workspace_bytes": ([U64, U64], ctypes.c_size_t),
            "zkl_hyrax_commit": ([P, P, U64, zkl_vec, U64, P, P], I32),
            "zkl_hyrax_prove_eval": ([P, zkl_vec, U64, U64, P, zkl_vec, P], I32),
            "zkl_matmul_prove": ([P, P, P, U64, U64, U64, P, P, P, zkl_vec, zkl_vec, P, P, P], I32),
            "zkl_ctx_wait": ([P], I32),
            "zkl_ctx_profile_read": ([P, ctypes.c_char_p, I32, ctypes.POINTER(ctypes.c_float),
                                      ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int), I32], I32),
            "zkl_vec_import": ([P, P, I32, zkl_vec, I64P], I32),
            "zkl_vec_import_i64": ([P, P, zkl_vec], I32),
            "zkl_vec_import_pair": ([P, P, P, ctypes.POINTER(zkl_fr), zkl_vec], I32),
            "zkl_vec_export": ([P, zkl_vec, P, I32], I32),
            "zkl_table_bytes": ([U64], ctypes.c_size_t),
            "zkl_table_create": ([P, zkl_vec, P, ctypes.c_size_t, ctypes.POINTER(P), I64P], I32),
            "zkl_table_destroy": ([P], None),
            "zkl_tlookup_prepare": ([P, zkl_vec, U64, P, P, I64P], I32),
            "zkl_tlookup_prepare_pair": ([P, P, P, ctypes.POINTER(zkl_fr), U64, P, zkl_vec, P, I64P], I32),
            "zkl_tlookup_prove": ([P, zkl_vec, U64, P, P, ctypes.POINTER(zkl_challenges), I32, zkl_vec, zkl_vec,
                                   ctypes.POINTER(zkl_fr), ctypes.POINTER(zkl_final_evals), I64P], I32),
            "zkl_tlookup_prove_fs": ([P, zkl_vec, U64, P, P, ctypes.c_char_p, I32, zkl_vec, zkl_vec,
                                      ctypes.POINTER(zkl_fr), ctypes.POINTER(zkl_final_evals), ctypes.POINTER(zkl_fr),
                                      I64P], I32),
            "zkl_tlookup_prove_p1": ([P, P, U64, P, P, U64, P, P, U64, ctypes.c_char_p, I32,
                                      ctypes.POINTER(zkl_p1_proof)], I32),
            "zkl_tlookup_prove_pair_host": ([P, P, P, U64, P, P, U64, ctypes.POINTER(zkl_fr),
                                             ctypes.POINTER(zkl_challenges), I32, ctypes.POINTER(zkl_fr),
                                             ctypes.POINTER(zkl_final_evals), P, I64P], I32),
            "zkl_sumcheck_prove": ([P, zkl_vec, zkl_vec, U64, zkl_vec, zkl_vec, zkl_vec,
                                    ctypes.POINTER(zkl_challenges), I32, ctypes.POINTER(zkl_fr),
                                    ctypes.POINTER(zkl_final_evals)], I32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


EXPORTED = ["zkl_strerror", "zkl_ctx_create", "zkl_nccl_unique_id", "zkl_ctx_create_dist", "zkl_ctx_destroy",
            "zkl_group_create", "zkl_group_destroy", "zkl_ctx_create_loopback",
            "zkl_last_error", "zkl_workspace_bytes", "zkl_ctx_set_workspace", "zkl_ctx_launch_count",
            "zkl_ctx_set_profiling", "zkl_ctx_profile_read", "zkl_ctx_set_async", "zkl_ctx_wait",
            "zkl_matmul_workspace_bytes", "zkl_matmul_prove",
            "zkl_table_attach_pair", "zkl_hyrax_pp_bytes", "zkl_hyrax_setup", "zkl_hyrax_export_generators", "zkl_hyrax_workspace_bytes",
            "zkl_hyrax_commit", "zkl_hyrax_prove_eval",
            "zkl_vec_import", "zkl_vec_import_i64", "zkl_vec_import_pair", "zkl_vec_export", "zkl_table_bytes",
            "zkl_table_create", "zkl_table_destroy", "zkl_tlookup_prepare", "zkl_tlookup_prepare_pair",
            "zkl_tlookup_prove", "zkl_tlookup_prove_fs", "zkl_tlookup_prove_pair_host",
            "zkl_tlookup_prove_p1", "zkl_sumcheck_prove"]


def __getattr__(name):   # C names exposed unchanged: zkl.zkl_tlookup_prove(...)
    if name in EXPORTED:
        return getattr(lib(), name)
    raise AttributeError(name)


# ---------------------------------------------------------------- marshalling helpers
def fr_from_int(x: int) -> zkl_fr:
    if not 0 <= x < R_MODULUS:
        raise ValueError("field element out of range")
    f = zkl_fr()
    for i in range(8):
        f.w[i] = (x >> (32 * i)) & 0xFFFFFFFF
    return f


def fr_to_int(f: zkl_fr) -> int:
    return sum(int(f.w[i]) << (32 * i) for i in range(8))


def ints_to_canon(xs: Sequence[int]) -> np.ndarray:
    """Python ints -> (n, 8) uint32 canonical little-endian words."""
    out = np.zeros((len(xs), 8), dtype=np.uint32)
    for i, x in enumerate(xs):
        for k in range(8):
            out[i, k] = (x >> (32 * k)) & 0xFFFFFFFF
    return out


def canon_to_ints(a: np.ndarray) -> List[int]:
    a = np.asarray(a, dtype=np.uint32).reshape(-1, 8).astype(object)
    return [int(sum(int(r[k]) << (32 * k) for k in range(8))) for r in a]


@dataclass
class Vec:
    """A device field vector: torch int32 storage of 8*n words (SoA Montgomery)."""
    data: "object"        # torch.Tensor
    n: int

    @property
    def c(self) -> zkl_vec:
        return zkl_vec(self.data.data_ptr() if self.data is not None else None, self.n)


@dataclass
class Proof:
    evals: List[List[int]]
    finals: Dict[str, int]
    A: Optional[Vec] = None
    B: Optional[Vec] = None


class Deferred:
    """Result of a call made in async mode (Context.set_async): filled in by Context.wait()."""

    def __init__(self, make):
        self._make, self._value, self.done = make, None, False

    def _resolve(self):
        self._value, self.done = self._make(), True

    def result(self):
        if not self.done:
            raise RuntimeError("not completed: call Context.wait() first")
        return self._value


class Context:
    """One device context: stream, workspace and the zkl_ctx handle."""

    def __init__(self, device: int = 0, stream=None, rank: int = 0, nranks: int = 1, nccl_id: bytes = None,
                 group: "LoopbackGroup" = None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("zkl needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = ctypes.c_void_p()
        if group is not None:
            nranks = group.nranks
            st = lib().zkl_ctx_create_loopback(device, ctypes.c_void_p(self.stream.cuda_stream), group.h, rank,
                                               ctypes.byref(h))
        elif nranks > 1:
            st = lib().zkl_ctx_create_dist(device, ctypes.c_void_p(self.stream.cuda_stream), nccl_id, rank, nranks,
                                           ctypes.byref(h))
        else:
            st = lib().zkl_ctx_create(device, ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h))
        if st:
            raise ZklError(st, -1, "context creation")
        self.h = h
        self.rank, self.nranks = rank, nranks
        self.ws = None
        self._tables = []
        self._async = False
        self._pending = []   # (err c_int64, Deferred or None) of calls enqueued in async mode

    def close(self):
        if getattr(self, "h", None):
            lib().zkl_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing
    def _check(self, st: int, idx: int = -1):
        if st:
            raise ZklError(st, idx, lib().zkl_last_error(self.h).decode(errors="replace"))

    @property
    def launches(self) -> int:
        return int(lib().zkl_ctx_launch_count(self.h))

    # -- async mode: K instances in flight = K contexts on K streams
    def set_async(self, on: bool):
        """In async mode prepare*/prove*/sumcheck enqueue and return at once; prove* return a Deferred."""
        self._check(lib().zkl_ctx_set_async(self.h, 1 if on else 0))
        self._async = bool(on)

    def _defer(self, err, make=None, keep=None):
        """`keep`: device buffers the library still reads at completion (e.g. prepare_pair's x, y for the range-miss
        fallback inside zkl_ctx_wait) -- referenced here until wait() so that temporaries are not freed early."""
        dfr = Deferred(make) if make is not None else None
        self._pending.append((err, dfr, keep))
        return dfr

    def wait(self):
        """Complete every call enqueued in async mode (raises the first error, in call order)."""
        st = lib().zkl_ctx_wait(self.h)
        pend, self._pending = self._pending, []
        if st:
            idx = next((e.value for e, _, _ in pend if e is not None and e.value != -1), -1)
            raise ZklError(st, idx, lib().zkl_last_error(self.h).decode(errors="replace"))
        for _, dfr, _ in pend:
            if dfr is not None:
                dfr._resolve()

    def set_profiling(self, on: bool):
        self._check(lib().zkl_ctx_set_profiling(self.h, 1 if on else 0))

    def profile_read(self, with_start: bool = False):
        """[(kernel name, ms[, start ms, stream tag])] of the launches recorded since profiling was (re)enabled
        or last read.  stream tag: 0 = ctx stream, 1 = table side, 2 = aux, 3 = async-mode histogram."""
        cap, nl = 256, 64
        names = ctypes.create_string_buffer(cap * nl)
        ms = (ctypes.c_float * cap)()
        st = (ctypes.c_float * cap)()
        tag = (ctypes.c_int * cap)()
        n = lib().zkl_ctx_profile_read(self.h, names, nl, ms, st, tag, cap)
        if n < 0:
            raise ZklError(-n, -1, "profile_read")
        raw = names.raw
        nm = [raw[i * nl:(i + 1) * nl].split(b"\0", 1)[0].decode() for i in range(n)]
        if with_start:
            return [(nm[i], float(ms[i]), float(st[i]), int(tag[i])) for i in range(n)]
        return [(nm[i], float(ms[i])) for i in range(n)]

    def reserve(self, D_local: int, N: int):
        need = int(lib().zkl_workspace_bytes(D_local, N, self.nranks))
        if need == 0:
            raise ZklError(2, -1, f"bad shape D_local={D_local} N={N}")
        self._ensure_ws(need)

    def _ensure_ws(self, need: int):
        if self.ws is None or self.ws.numel() < need + 256:
            self.ws = None
            self.torch.cuda.synchronize(self.device)
            self.torch.cuda.empty_cache()
            self.ws = self.torch.empty(need + 256, dtype=self.torch.uint8, device=self.device)
        ptr = self.ws.data_ptr()
        pad = (-ptr) % 256
        self._check(lib().zkl_ctx_set_workspace(self.h, ctypes.c_void_p(ptr + pad), self.ws.numel() - pad))

    def vec(self, n: int) -> Vec:
        return Vec(self.torch.empty(max(8 * n, 32), dtype=self.torch.int32, device=self.device), n)

    # -- a1
    def import_canon(self, canon: np.ndarray, dst: Optional[Vec] = None) -> Vec:
        canon = np.ascontiguousarray(canon, dtype=np.uint32).reshape(-1, 8)
        n = canon.shape[0]
        dst = dst or self.vec(n)
        err = ctypes.c_int64(-1)
        st = lib().zkl_vec_import(self.h, canon.ctypes.data, 0, dst.c, ctypes.byref(err))
        self._check(st, err.value)
        return dst

    def import_canon_device(self, canon_dev, n: int, dst: Optional[Vec] = None) -> Vec:
        dst = dst or self.vec(n)
        err = ctypes.c_int64(-1)
        st = lib().zkl_vec_import(self.h, ctypes.c_void_p(canon_dev.data_ptr()), 1, dst.c, ctypes.byref(err))
        self._check(st, err.value)
        return dst

    def import_ints(self, x, dst: Optional[Vec] = None) -> Vec:
        t = self.torch.as_tensor(np.asarray(x, dtype=np.int64)).to(self.device) if not hasattr(x, "data_ptr") else x
        n = t.numel()
        dst = dst or self.vec(n)
        self._check(lib().zkl_vec_import_i64(self.h, ctypes.c_void_p(t.data_ptr()), dst.c))
        return dst

    def import_pair(self, x, y, alpha_f: int, dst: Optional[Vec] = None) -> Vec:
        tx = x if hasattr(x, "data_ptr") else self.torch.as_tensor(np.asarray(x, np.int32)).to(self.device)
        ty = y if hasattr(y, "data_ptr") else self.torch.as_tensor(np.asarray(y, np.int32)).to(self.device)
        n = tx.numel()
        dst = dst or self.vec(n)
        af = fr_from_int(alpha_f % R_MODULUS)
        self._check(lib().zkl_vec_import_pair(self.h, ctypes.c_void_p(tx.data_ptr()), ctypes.c_void_p(ty.data_ptr()),
                                              ctypes.byref(af), dst.c))
        return dst

    def export(self, v: Vec) -> np.ndarray:
        out = np.zeros((v.n, 8), dtype=np.uint32)
        self._check(lib().zkl_vec_export(self.h, v.c, out.ctypes.data, 0))
        return out

    def export_ints(self, v: Vec) -> List[int]:
        return canon_to_ints(self.export(v))

    # -- a2
    def table_mem(self, N: int):
        return self.torch.empty(int(lib().zkl_table_bytes(N)) + 256, dtype=self.torch.uint8, device=self.device)

    def table(self, T: Vec, mem=None):
        nbytes = int(lib().zkl_table_bytes(T.n))
        mem = mem if mem is not None else self.table_mem(T.n)
        ptr = mem.data_ptr()
        pad = (-ptr) % 256
        h = ctypes.c_void_p()
        err = ctypes.c_int64(-1)
        st = lib().zkl_table_create(self.h, T.c, ctypes.c_void_p(ptr + pad), nbytes, ctypes.byref(h),
                                    ctypes.byref(err))
        self._check(st, err.value)
        tab = Table(h, T.n, mem, self)
        return tab

    def table_attach_pair(self, tab: "Table", tx, ty, alpha_f: int) -> bool:
        """Declare T_j = tx_j + alpha_f ty_j with tx a contiguous range (the function-lookup fast path of
        prepare_pair).  Returns False (and the table keeps the hash index only) if T is not of that form."""
        ttx = tx if hasattr(tx, "data_ptr") else self.torch.as_tensor(np.asarray(tx, np.int32)).to(self.device)
        tty = ty if hasattr(ty, "data_ptr") else self.torch.as_tensor(np.asarray(ty, np.int32)).to(self.device)
        af = fr_from_int(alpha_f % R_MODULUS)
        st = lib().zkl_table_attach_pair(self.h, tab.h, ctypes.c_void_p(ttx.data_ptr()), ctypes.c_void_p(tty.data_ptr()),
                                         ctypes.byref(af))
        if st == 1:   # E_ARG: not a pair-range table
            return False
        self._check(st)
        return True

    # -- a3
    def prepare(self, S: Vec, D: int, tab: "Table", m=None):
        m = m if m is not None else self.torch.empty(tab.N, dtype=self.torch.int32, device=self.device)
        err = ctypes.c_int64(-1)
        st = lib().zkl_tlookup_prepare(self.h, S.c, D, tab.h, ctypes.c_void_p(m.data_ptr()), ctypes.byref(err))
        self._check(st, err.value)
        if self._async:
            self._defer(err)
        return m

    def prepare_pair(self, x, y, alpha_f: int, D: int, tab: "Table", S: Optional[Vec] = None, m=None,
                     virtual_s: bool = False):
        """a1 + a3 fused for function lookups: S = x + alpha_f y is written to S and counted into m.
        virtual_s: S is not materialised (only the table keys are kept; prove(None, ...) gathers S_i = T_key);
        returns (None, m)."""
        tx = x if hasattr(x, "data_ptr") else self.torch.as_tensor(np.asarray(x, np.int32)).to(self.device)
        ty = y if hasattr(y, "data_ptr") else self.torch.as_tensor(np.asarray(y, np.int32)).to(self.device)
        S = Vec(None, tx.numel()) if virtual_s else (S or self.vec(tx.numel()))
        m = m if m is not None else self.torch.empty(tab.N, dtype=self.torch.int32, device=self.device)
        af = fr_from_int(alpha_f % R_MODULUS)
        err = ctypes.c_int64(-1)
        st = lib().zkl_tlookup_prepare_pair(self.h, ctypes.c_void_p(tx.data_ptr()), ctypes.c_void_p(ty.data_ptr()),
                                            ctypes.byref(af), D, tab.h, S.c, ctypes.c_void_p(m.data_ptr()),
                                            ctypes.byref(err))
        self._check(st, err.value)
        if self._async:
            self._defer(err, keep=(tx, ty))
        return (None if virtual_s else S), m

    # -- a4..a9
    @staticmethod
    def challenges(beta: int, alpha1: int, alpha2: int, u: Sequence[int], r: Sequence[int]):
        U = (zkl_fr * max(len(u), 1))(*[fr_from_int(x % R_MODULUS) for x in u])
        Rr = (zkl_fr * max(len(r), 1))(*[fr_from_int(x % R_MODULUS) for x in r])
        ch = zkl_challenges(fr_from_int(beta % R_MODULUS), fr_from_int(alpha1 % R_MODULUS),
                            fr_from_int(alpha2 % R_MODULUS), ctypes.cast(U, ctypes.POINTER(zkl_fr)),
                            ctypes.cast(Rr, ctypes.POINTER(zkl_fr)))
        ch._keep = (U, Rr)
        return ch

    def prove(self, S: Optional[Vec], D: int, tab: "Table", m, ch, variant: int = PAPER, want_A: bool = False,
              want_B: bool = False) -> Proof:
        """S None: the virtual S of the preceding prepare_pair(..., virtual_s=True) on this context."""
        S = S if S is not None else Vec(None, D // self.nranks)
        d = D.bit_length() - 1
        A = self.vec(S.n) if want_A else Vec(None, S.n)
        B = self.vec(tab.N) if want_B else Vec(None, tab.N)
        evals = (zkl_fr * (4 * max(d, 1)))()
        fin = zkl_final_evals()
        err = ctypes.c_int64(-1)
        st = lib().zkl_tlookup_prove(self.h, S.c, D, tab.h, ctypes.c_void_p(m.data_ptr()), ctypes.byref(ch), variant,
                                     A.c, B.c, evals, ctypes.byref(fin), ctypes.byref(err))
        self._check(st, err.value)
        make = lambda: Proof(_evals(evals, d), _finals(fin), A if want_A else None, B if want_B else None)  # noqa: E731
        if self._async:
            return self._defer(err, make)
        return make()

    def prove_pair_host(self, x, y, tx, ty, alpha_f: int, D: int, ch, variant: int = PAPER, want_m: bool = False):
        """The end-to-end step from HOST int32 buffers (numpy arrays or CPU torch tensors, ideally pinned):
        zkl_tlookup_prove_pair_host copies them into context-owned device memory, builds the table and proves with a
        virtual S.  Returns Proof (and m as a numpy array if want_m)."""
        def hptr(a):
            if hasattr(a, "data_ptr"):
                assert not a.is_cuda and a.dtype == self.torch.int32 and a.is_contiguous()
                return ctypes.c_void_p(a.data_ptr()), a.numel()
            a = np.ascontiguousarray(a, dtype=np.int32)
            hptr.keep.append(a)
            return ctypes.c_void_p(a.ctypes.data), a.size
        hptr.keep = []
        (px, nx), (py, _), (ptx, N), (pty, _) = hptr(x), hptr(y), hptr(tx), hptr(ty)
        d = D.bit_length() - 1
        evals = (zkl_fr * (4 * max(d, 1)))()
        fin = zkl_final_evals()
        err = ctypes.c_int64(-1)
        af = fr_from_int(alpha_f % R_MODULUS)
        mh = np.zeros(N, dtype=np.uint32) if want_m else None
        st = lib().zkl_tlookup_prove_pair_host(self.h, px, py, D, ptx, pty, N, ctypes.byref(af), ctypes.byref(ch),
                                               variant, evals, ctypes.byref(fin),
                                               ctypes.c_void_p(mh.ctypes.data) if want_m else None, ctypes.byref(err))
        self._check(st, err.value)
        pf = Proof(_evals(evals, d), _finals(fin))
        return (pf, mh) if want_m else pf

    def prove_p1(self, pp, x, y, tx, ty, seed: bytes, variant: int = PAPER):
        """Protocol 1 with its commitments (zkl_tlookup_prove_p1): x, y, tx, ty int32 (device tensors or arrays).
        Returns the proof in the form oracle/protocol1.py verifies (points as (x, y) or None, field elements as
        ints)."""
        dev = lambda a: a if hasattr(a, "data_ptr") else self.torch.as_tensor(np.asarray(a, np.int32)).to(self.device)  # noqa: E731
        xd, yd, txd, tyd = dev(x), dev(y), dev(tx), dev(ty)
        D, N, cols = xd.numel(), txd.numel(), pp["cols"]
        d = D.bit_length() - 1
        rD, rN = D // cols, N // cols
        arr = {k: (zkl_g1 * (rD if k in ("C_X", "C_Y", "C_A") else rN))() for k in
               ("C_X", "C_Y", "C_TX", "C_TY", "C_m", "C_A", "C_B")}
        wv = {k: (zkl_fr * cols)() for k in ("w_A", "w_X", "w_Y", "w_TX", "w_TY", "w_m", "w_B")}
        ev = (zkl_fr * (4 * d))()
        der = (zkl_fr * (3 + 2 * d))()
        pf = zkl_p1_proof()
        for k, a in arr.items():
            setattr(pf, k, ctypes.cast(a, _G1P))
        for k, a in wv.items():
            setattr(pf, k, ctypes.cast(a, _FRP))
        pf.round_evals = ctypes.cast(ev, _FRP)
        pf.derived = ctypes.cast(der, _FRP)
        if len(seed) != 32:
            raise ValueError("seed must be 32 bytes")
        self._check(lib().zkl_tlookup_prove_p1(self.h, ctypes.c_void_p(pp["ptr"]), cols, ctypes.c_void_p(xd.data_ptr()),
                                               ctypes.c_void_p(yd.data_ptr()), D, ctypes.c_void_p(txd.data_ptr()),
                                               ctypes.c_void_p(tyd.data_ptr()), N, seed, variant, ctypes.byref(pf)))
        dv = [fr_to_int(der[i]) for i in range(3 + 2 * d)]
        C = {k[2:]: [g1_to_py(a[i]) for i in range(len(a))] for k, a in arr.items()}
        proofs = {k[2:]: ([fr_to_int(wv[k][i]) for i in range(cols)], fr_to_int(getattr(pf, "y_" + k[2:])))
                  for k in wv}
        return {"D": D, "N": N, "cols": cols, "variant": variant, "seed": seed, "C": C,
                "alpha_f": fr_to_int(pf.alpha_f), "evals": _evals(ev, d), "finals": _finals(pf.finals),
                "derived": {"beta": dv[0], "alpha1": dv[1], "alpha2": dv[2], "u": dv[3:3 + d], "r": dv[3 + d:]},
                "eval_proofs": proofs}

    def prove_fs(self, S: Vec, D: int, tab: "Table", m, seed: bytes, variant: int = PAPER, want_A: bool = False,
                 want_B: bool = False):
        """Fiat-Shamir prove: challenges derived on the device from a SHA-256 transcript seeded by `seed` (32 B).
        Returns (Proof, derived) with derived = dict(beta, alpha1, alpha2, u, r) (canonical ints)."""
        if len(seed) != 32:
            raise ValueError("seed must be 32 bytes")
        S = S if S is not None else Vec(None, D // self.nranks)
        d = D.bit_length() - 1
        A = self.vec(S.n) if want_A else Vec(None, S.n)
        B = self.vec(tab.N) if want_B else Vec(None, tab.N)
        evals = (zkl_fr * (4 * max(d, 1)))()
        der = (zkl_fr * (3 + 2 * max(d, 1)))()
        fin = zkl_final_evals()
        err = ctypes.c_int64(-1)
        st = lib().zkl_tlookup_prove_fs(self.h, S.c, D, tab.h, ctypes.c_void_p(m.data_ptr()), seed, variant, A.c,
                                        B.c, evals, ctypes.byref(fin), der, ctypes.byref(err))
        self._check(st, err.value)

        def make():
            dv = [fr_to_int(der[i]) for i in range(3 + 2 * d)]
            derived = {"beta": dv[0], "alpha1": dv[1], "alpha2": dv[2], "u": dv[3:3 + d], "r": dv[3 + d:3 + 2 * d]}
            return Proof(_evals(evals, d), _finals(fin), A if want_A else None, B if want_B else None), derived
        if self._async:
            return self._defer(err, make)
        return make()

    def sumcheck(self, A: Vec, S: Vec, D: int, B: Vec, T: Vec, mfr: Vec, ch, variant: int = PAPER) -> Proof:
        d = D.bit_length() - 1
        evals = (zkl_fr * (4 * max(d, 1)))()
        fin = zkl_final_evals()
        st = lib().zkl_sumcheck_prove(self.h, A.c, S.c, D, B.c, T.c, mfr.c, ctypes.byref(ch), variant, evals,
                                      ctypes.byref(fin))
        self._check(st)
        make = lambda: Proof(_evals(evals, d), _finals(fin))  # noqa: E731
        if self._async:
            return self._defer(None, make)
        return make()

    # -- f4: matmul sumcheck
    def matmul_prove(self, A, B, u: Sequence[int], v: Sequence[int], r: Sequence[int], want_ab: bool = False):
        """Sumcheck of C~(u, v) = sum_i A~(u, i) B~(i, v) for int32 A (m x n), B (n x p) (torch device tensors or
        arrays).  Returns dict(claim, evals [[g_k(0), g_k(1), g_k(2)]...], finals [a~(w), b~(w)], a, b)."""
        tA = A if hasattr(A, "data_ptr") else self.torch.as_tensor(np.asarray(A, np.int32)).to(self.device)
        tB = B if hasattr(B, "data_ptr") else self.torch.as_tensor(np.asarray(B, np.int32)).to(self.device)
        if tA.dtype != self.torch.int32 or tB.dtype != self.torch.int32 or tA.dim() != 2 or tB.dim() != 2:
            raise ValueError("A, B: 2-D int32")
        tA, tB = tA.contiguous(), tB.contiguous()
        m, n = tA.shape
        n2, p = tB.shape
        if n != n2:
            raise ValueError("inner dimensions differ")
        need = int(lib().zkl_matmul_workspace_bytes(m, n, p))
        if need == 0:
            raise ZklError(2, -1, f"bad shape m={m} n={n} p={p}")
        self._ensure_ws(need)
        L = n.bit_length() - 1
        U = (zkl_fr * max(len(u), 1))(*[fr_from_int(x % R_MODULUS) for x in u])
        V = (zkl_fr * max(len(v), 1))(*[fr_from_int(x % R_MODULUS) for x in v])
        Rr = (zkl_fr * max(len(r), 1))(*[fr_from_int(x % R_MODULUS) for x in r])
        a = self.vec(n) if want_ab else Vec(None, n)
        b = self.vec(n) if want_ab else Vec(None, n)
        claim = zkl_fr()
        ev = (zkl_fr * (3 * max(L, 1)))()
        fin = (zkl_fr * 2)()
        st = lib().zkl_matmul_prove(self.h, ctypes.c_void_p(tA.data_ptr()), ctypes.c_void_p(tB.data_ptr()), m, n, p,
                                    U, V, Rr, a.c, b.c, ctypes.byref(claim), ev, fin)
        self._check(st)
        return {"claim": fr_to_int(claim), "evals": [[fr_to_int(ev[3 * k + t]) for t in range(3)] for k in range(L)],
                "finals": [fr_to_int(fin[0]), fr_to_int(fin[1])], "a": a if want_ab else None,
                "b": b if want_ab else None}

    # -- f3: Hyrax / Pedersen commitments
    def hyrax_setup(self, cols: int):
        """Public parameters for rows of `cols` entries: G_0..G_{cols-1}, H and their window tables (device)."""
        nb = int(lib().zkl_hyrax_pp_bytes(cols))
        if nb == 0:
            raise ZklError(2, -1, f"bad cols {cols}")
        pp = self.torch.empty(nb + 256, dtype=self.torch.uint8, device=self.device)
        pad = (-pp.data_ptr()) % 256
        self._check(lib().zkl_hyrax_setup(self.h, cols, ctypes.c_void_p(pp.data_ptr() + pad), nb))
        return {"cols": cols, "mem": pp, "ptr": pp.data_ptr() + pad}

    def hyrax_generators(self, pp):
        out = (zkl_g1 * (pp["cols"] + 1))()
        self._check(lib().zkl_hyrax_export_generators(self.h, ctypes.c_void_p(pp["ptr"]), pp["cols"], out))
        pts = [g1_to_py(out[i]) for i in range(pp["cols"] + 1)]
        return pts[:-1], pts[-1]

    def hyrax_commit(self, pp, S: Vec, D: int, rho: Optional[Sequence[int]] = None):
        cols = pp["cols"]
        need = int(lib().zkl_hyrax_workspace_bytes(D, cols))
        if need == 0:
            raise ZklError(2, -1, f"bad shape D={D} cols={cols}")
        self._ensure_ws(need)
        rows = D // cols
        rh = None
        if rho is not None:
            rh = (zkl_fr * rows)(*[fr_from_int(x % R_MODULUS) for x in rho])
        out = (zkl_g1 * rows)()
        self._check(lib().zkl_hyrax_commit(self.h, ctypes.c_void_p(pp["ptr"]), cols, S.c, D, rh, out))
        return [g1_to_py(out[j]) for j in range(rows)]

    def hyrax_prove_eval(self, S: Vec, D: int, cols: int, v: Sequence[int]):
        need = int(lib().zkl_hyrax_workspace_bytes(D, cols))
        if need == 0:
            raise ZklError(2, -1, f"bad shape D={D} cols={cols}")
        self._ensure_ws(need)
        V = (zkl_fr * max(len(v), 1))(*[fr_from_int(x % R_MODULUS) for x in v])
        w = self.vec(cols)
        y = zkl_fr()
        self._check(lib().zkl_hyrax_prove_eval(self.h, S.c, D, cols, V, w.c, ctypes.byref(y)))
        return w, fr_to_int(y)


class Table:
    def __init__(self, h, N, mem, ctx):
        self.h, self.N, self.mem, self.ctx = h, N, mem, ctx

    def __del__(self):
        try:
            if self.h:
                lib().zkl_table_destroy(self.h)
                self.h = None
        except Exception:
            pass


def _evals(arr, d) -> List[List[int]]:
    return [[fr_to_int(arr[4 * k + t]) for t in range(4)] for k in range(d)]


def _finals(f: zkl_final_evals) -> Dict[str, int]:
    return {"A": fr_to_int(f.A), "S": fr_to_int(f.S), "B": fr_to_int(f.B), "T": fr_to_int(f.T),
            "m": fr_to_int(f.m)}


class LoopbackGroup:
    """P virtual ranks on one device (zkl_group_create); one Context(group=..., rank=p) per host thread."""

    def __init__(self, nranks: int, device: int = 0, max_D_local: int = 1 << 20, max_N: int = 1 << 16):
        h = ctypes.c_void_p()
        st = lib().zkl_group_create(device, nranks, max_D_local, max_N, ctypes.byref(h))
        if st:
            raise ZklError(st, -1, "zkl_group_create")
        self.h, self.nranks = h, nranks

    def close(self):
        if self.h:
            lib().zkl_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = lib().zkl_nccl_unique_id(buf)
    if st:
        raise ZklError(st, -1, "ncclGetUniqueId")
    return buf.raw
