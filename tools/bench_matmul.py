"""Matmul sumcheck at LLaMA-2-7B projection shapes on one B200.

    python tools/bench_matmul.py [tokens]      (default 2048)

Per shape: device time of one proof (restrictions + sumcheck; inputs resident in HBM; CUDA events, warm-up 3),
the kernel breakdown from the library's event profiler, and the restriction kernels' HBM rate against the measured
copy bandwidth (they read A and B once, 4 B per int32 entry).  One JSON line per shape; a last line times the
Python oracle on a bounded sample (entries per second of the restriction by its definition).
"""
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2404_16109_b200 import zkl  # noqa: E402

R = zkl.R_MODULUS


def peak_hbm():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        for k in ("hbm_gbps", "hbm_GBps", "hbm"):
            if k in d:
                v = d[k]
                return float(v["value"] if isinstance(v, dict) else v)
    except Exception:
        pass
    return 6555.5


def main():
    tokens = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    dev = torch.device("cuda", 0)
    ctx = zkl.Context(0)
    rng = random.Random(1)
    shapes = [("attn q/k/v/o", tokens, 4096, 4096), ("ffn up/gate (11008 -> 16384)", tokens, 4096, 16384),
              ("ffn down", tokens, 16384, 4096)]
    hbm = peak_hbm()
    for name, m, n, p in shapes:
        g = torch.Generator(device=dev).manual_seed(7)
        A = torch.randint(-(1 << 15), 1 << 15, (m, n), dtype=torch.int32, device=dev, generator=g)
        B = torch.randint(-(1 << 15), 1 << 15, (n, p), dtype=torch.int32, device=dev, generator=g)
        u = [rng.randrange(R) for _ in range(m.bit_length() - 1)]
        v = [rng.randrange(R) for _ in range(p.bit_length() - 1)]
        r = [rng.randrange(R) for _ in range(n.bit_length() - 1)]
        for _ in range(3):
            ctx.matmul_prove(A, B, u, v, r)
        torch.cuda.synchronize()
        steps = 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        for _ in range(steps):
            ctx.matmul_prove(A, B, u, v, r)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        ctx.set_profiling(True)
        ctx.matmul_prove(A, B, u, v, r)
        prof = ctx.profile_read()
        ctx.set_profiling(False)
        kern = {}
        for nm, t in prof:
            kern[nm] = kern.get(nm, 0.0) + t
        restrict_ms = sum(v for k, v in kern.items() if k.startswith("k_mm_restrict") or k == "k_mm_sum_chunks")
        rbytes = 4 * (m * n + n * p)
        print(json.dumps({"shape": name, "m": m, "n": n, "p": p, "ms_per_proof": ms,
                          "entries_per_s": (m * n + n * p) / (ms / 1e3),
                          "restrict_ms": restrict_ms, "restrict_GBps": rbytes / (restrict_ms / 1e3) / 1e9 if restrict_ms else None,
                          "hbm_peak_GBps": hbm, "restrict_frac_of_hbm": (rbytes / (restrict_ms / 1e3) / 1e9 / hbm) if restrict_ms else None,
                          "kernels_ms": {k: round(v, 4) for k, v in sorted(kern.items(), key=lambda x: -x[1])}}), flush=True)
        del A, B
        torch.cuda.empty_cache()
    # oracle (the definition, Python big integers) on a bounded sample
    sys.path.insert(0, ROOT)
    from oracle import matmul as MM
    m, n, p = 8, 256, 8
    A = [[rng.randrange(-(1 << 15), 1 << 15) for _ in range(n)] for _ in range(m)]
    B = [[rng.randrange(-(1 << 15), 1 << 15) for _ in range(p)] for _ in range(n)]
    t0 = time.perf_counter()
    MM.prove(MM.field_matrix(A), MM.field_matrix(B), [rng.randrange(R) for _ in range(3)],
             [rng.randrange(R) for _ in range(3)], [rng.randrange(R) for _ in range(8)])
    dt = time.perf_counter() - t0
    print(json.dumps({"oracle": "oracle/matmul.py prove (Python, 1 core)", "m": m, "n": n, "p": p, "s": dt,
                      "entries_per_s": (m * n + n * p) / dt}))


if __name__ == "__main__":
    main()
