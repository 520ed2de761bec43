"""Write the full-size parity goldens tests/golden/<cfg>.json from the CPU oracle.

Imports only `oracle/` (the streaming C tier, zko_tlookup_pair_stream) and `workloads/` (the seeded input
generator): no value here comes from the CUDA path.  Each golden holds the SHA-256 of the generated integer inputs
(so generator drift is detected before any comparison), the digests of m (u32 LE) and B (32-byte canonical LE per
entry), every round polynomial g_k(0..3) and the five final evaluations, as hex.

    python tools/make_goldens.py H 3 4.0 4.1 4.2 4.3 4.4 5      # all (C5 takes ~10-20 min on 8 cores)

Configurations (BASELINE.json configs):
  H    activation (SiLU) D = 2^26 into N = 2^16, PAPER variant (the bench workload)
  3    activation (SiLU) 2048 x 11008 zero-padded to 2^25, LOGUP variant
  4.k  zkAttn digit instance k (0..4) at the full 32 heads x 2048 x 2048 = 2^27, PAPER variant
  5    activation (SiLU) D = 2^30, PAPER variant (inputs drawn in 2^26 chunks)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from oracle import c_oracle as C  # noqa: E402
from oracle import tlookup as TL  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def pair_inputs(cfg: str):
    """(x, y, tx, ty, challenges, variant, meta) of a configuration, all as int32 pair form."""
    if cfg in ("H", "3"):
        wl = W.activation(cfg)
        variant = TL.PAPER if cfg == "H" else TL.LOGUP
        return wl.x, wl.y, wl.tx, wl.ty, wl.chal, variant, {"real": wl.meta["real"], "fn": wl.meta["fn"]}
    if cfg == "5":
        D = 1 << 30
        tx, ty = W.activation_table("silu")
        x = np.empty(D, dtype=np.int32)
        chunk = 1 << 26
        for start in range(0, D, chunk):
            x[start:start + chunk] = W.activation_x("5", start, chunk, D)
        y = ty[x.astype(np.int64) + 32768].astype(np.int32)
        return x, y, tx.astype(np.int32), ty.astype(np.int32), W.challenges("5", 30), TL.PAPER, {"real": D, "fn": "silu"}
    if cfg.startswith("4."):
        k = int(cfg.split(".")[1])
        wl = W.zkattn_digits(k, heads=32)
        if wl.kind == "int":   # range instance: S = x + alpha_f * 0, T = [0, 2^16)
            x = wl.s.astype(np.int32)
            return (x, np.zeros_like(x), wl.t.astype(np.int32), np.zeros(wl.N, np.int32), wl.chal, TL.PAPER,
                    {"kind": "range"})
        return wl.x, wl.y, wl.tx, wl.ty, wl.chal, TL.PAPER, {"kind": "function"}
    raise ValueError(cfg)


def make(cfg: str, s: int = None) -> dict:
    t0 = time.time()
    x, y, tx, ty, ch, variant, meta = pair_inputs(cfg)
    D, N = x.shape[0], tx.shape[0]
    d = D.bit_length() - 1
    s = s if s is not None else (4 if d >= 30 else 2)
    tgen = time.time() - t0
    chal = C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
    t1 = time.time()
    res = C.prove_pair_stream(x, y, tx, ty, ch.alpha_f, chal, variant, s)
    tor = time.time() - t1
    assert int(res.m.astype(np.int64).sum()) == D
    Bc = np.ascontiguousarray(res.B, dtype=np.uint64)
    out = {
        "config": cfg, "D": D, "N": N, "variant": "paper" if variant == TL.PAPER else "logup",
        "inputs_sha256": {"x": sha(x.astype("<i4")), "y": sha(y.astype("<i4")), "tx": sha(tx.astype("<i4")),
                          "ty": sha(ty.astype("<i4"))},
        "alpha_f": hex(ch.alpha_f % C.R),
        "m_sha256": sha(res.m.astype("<u4")),
        "B_sha256": sha(Bc.astype("<u8")),
        "evals": [[hex(v) for v in g] for g in res.evals],
        "finals": {k: hex(v) for k, v in res.finals.items()},
        "meta": meta,
        "generated_by": "tools/make_goldens.py (oracle/c zko_tlookup_pair_stream, s = %d)" % s,
        "oracle_seconds": round(tor, 1), "generator_seconds": round(tgen, 1), "threads": C.num_threads(),
    }
    return out


def main(cfgs):
    os.makedirs(GOLDEN, exist_ok=True)
    for cfg in cfgs:
        g = make(cfg)
        path = os.path.join(GOLDEN, f"full_{cfg}.json")
        with open(path, "w") as f:
            json.dump(g, f, indent=1)
        print(f"{cfg}: D=2^{g['D'].bit_length() - 1} oracle {g['oracle_seconds']} s -> {path}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["H"])
