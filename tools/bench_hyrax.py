"""Hyrax commitment throughput on one B200.

    python tools/bench_hyrax.py [log2D ...]      (default 16 18 20)

Per D (cols = 2^ceil(log2(D)/2)): setup time (generators + tables, once per cols), commit time of a random S
(CUDA events around the call, warm-up 1), the kernel breakdown, and the achieved rate of G1 mixed additions and F_q
multiplications in the dominant kernel (64 windowed additions per scalar, 4 doublings per window and 16-column slice;
11 F_q muls per mixed addition, 7 per doubling).  The Python oracle's rate (scalar multiplications by definition) on
a bounded sample closes the output.
"""
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2404_16109_b200 import zkl  # noqa: E402

R = zkl.R_MODULUS


def main():
    logs = [int(a) for a in sys.argv[1:]] or [16, 18, 20]
    ctx = zkl.Context(0)
    rng = random.Random(1)
    for ld in logs:
        D = 1 << ld
        cols = 1 << ((ld + 1) // 2)
        t0 = time.perf_counter()
        pp = ctx.hyrax_setup(cols)
        setup_s = time.perf_counter() - t0
        S = ctx.vec(D)
        # random canonical S on the device (imported in chunks)
        import numpy as np
        npr = np.random.default_rng(ld)
        canon = npr.integers(0, 1 << 32, size=(D, 8), dtype=np.uint64).astype(np.uint32)
        canon[:, 7] &= 0x3FFFFFFF   # < 2^254 < r
        ctx.import_canon(canon, dst=S)
        ctx.hyrax_commit(pp, S, D)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        C = ctx.hyrax_commit(pp, S, D)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ctx.set_profiling(True)
        ctx.hyrax_commit(pp, S, D)
        prof = dict(ctx.profile_read())
        ctx.set_profiling(False)
        kms = prof.get("k_hx_commit_partial", 0.0)
        adds = D * 64 * 15 / 16                      # nonzero 4-bit digits on average
        dbls = (D // 16) * 8 * 7 * 4                 # per (16-column slice, chunk): 7 x 4 doublings
        fq_muls = adds * 11 + dbls * 7
        print(json.dumps({"D": D, "rows": D // cols, "cols": cols, "setup_s": setup_s, "commit_ms": ms,
                          "elements_per_s": D / (ms / 1e3), "kernels_ms": prof,
                          "g1_adds_per_s": adds / (kms / 1e3) if kms else None,
                          "fq_muls_per_s": fq_muls / (kms / 1e3) if kms else None,
                          "commitment_bytes": len(C) * 96}), flush=True)
    from oracle import hyrax as HX
    G, Hb = HX.generators(4)
    sc = [rng.randrange(R) for _ in range(8)]
    t0 = time.perf_counter()
    HX.commit(sc, 4, G, Hb)
    dt = time.perf_counter() - t0
    print(json.dumps({"oracle": "oracle/hyrax.py commit (Python, 1 core)", "elements": 8, "s": dt,
                      "elements_per_s": 8 / dt}))


if __name__ == "__main__":
    main()
