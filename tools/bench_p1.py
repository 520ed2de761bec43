"""Time Protocol 1 with its commitments (zkl_tlookup_prove_p1) at a few sizes on one GPU: the whole non-interactive
proof (Hyrax commitments of T_X, T_Y, X, Y, m, A, B, the transcript, the sumcheck, seven proofs of evaluation).

    python tools/bench_p1.py [log2D ...]        (N = 2^16 SiLU table, rows of 2^10; profiles/r02_p1.jsonl)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2404_16109_b200 import zkl  # noqa: E402


def main(logs):
    ctx = zkl.Context(0)
    dev = torch.device("cuda", 0)
    cols = 1 << 10
    pp = ctx.hyrax_setup(cols)
    for ld in logs:
        wl = W.activation("H", D=1 << ld)
        ctx.reserve(wl.D, wl.N)
        xd, yd = torch.from_numpy(wl.x).to(dev), torch.from_numpy(wl.y).to(dev)
        txd, tyd = torch.from_numpy(wl.tx).to(dev), torch.from_numpy(wl.ty).to(dev)
        ctx.prove_p1(pp, xd, yd, txd, tyd, bytes(32), zkl.PAPER)   # warm-up (allocates the owned buffers)
        torch.cuda.synchronize()
        ctx.set_profiling(True)
        t0 = time.perf_counter()
        ctx.prove_p1(pp, xd, yd, txd, tyd, bytes(32), zkl.PAPER)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        kern = {}
        for name, ms in ctx.profile_read():
            kern[name] = kern.get(name, 0.0) + ms
        ctx.set_profiling(False)
        top = dict(sorted(kern.items(), key=lambda kv: -kv[1])[:8])
        print(json.dumps({"D": wl.D, "N": wl.N, "cols": cols, "seconds": wall, "lookups_per_s": wl.D / wall,
                          "top_kernels_ms": {k: round(v, 3) for k, v in top.items()}}), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [16, 18, 20])
