#!/usr/bin/env python
"""bench.py — tlookup lookups/s (bit-exact proof) at D = 2^26 on 1..8 B200s, with % of roofline.

Contract (driver): `python bench.py --gpus N --steps K --warmup W`; for N > 1 launched under torchrun
(one rank per GPU, NCCL).  Rank 0 prints ONE JSON line.

A step is one pass of the whole hot path over the workload H
(LLaMA-2 SwiGLU/SiLU activation tlookup, D = 2^26 lookups into the N = 2^16 function table):
  a1 import  T = T_X + alpha_f T_Y, a2 table handle (validation + hash index),
  a1 + a3 zkl_tlookup_prepare_pair: S = X + alpha_f Y from the int32 tensors resident in HBM, fused with
          the index map, then the multiplicities m,
  a4-a9 zkl_tlookup_prove (A, B, the 26-round sumcheck, finals) — transcript returned to the host.
Under P ranks the D = 2^26 lookups are split over the ranks on the top log2 P hypercube variables
(strong scaling); value = D / max-over-ranks step time.

`--impl reference` times the CPU oracle (oracle/c, the streaming C tier, as it stands) on the full workload H
(2^26 lookups, ~20-30 s per run) on the host cores, rank 0 only; warm-up runs use a 2^16 sample.

Roofline: the path is bound by the integer multiply pipe.  peak = the measured IMAD.WIDE rate
(MEASURED_INT_PEAKS.json, tools/microbench_int.cu) / 112 products per 8x32-bit Montgomery multiplication; the
dominant kernel's achieved rate counts 8 Fr multiplications per new pair over the launches that ran; the whole
step counts 5 per lookup (round 1: 2 per pair; rounds >= 2: 8 per pair, sum 4 per lookup) + 16 per table entry.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "tlookup lookups/sec (bit-exact proof) at D=2^26 on 1/2/4/8 B200; % roofline"
UNIT = "lookups/s"
WORKLOAD = "H: LLaMA-2 SwiGLU (SiLU) activation tlookup, D=2^26 lookups into an N=2^16 function table"
# ALU roofline: the measured IMAD.WIDE.U32 rate x 148 SMs x 1965 MHz / 112 products per Montgomery
# multiplication (64 operand + 48 reduction products: r0 = 1 and r1 = 2^32 - 1 need none).
SMS, MAX_MHZ, PRODUCTS_PER_MUL = 148, 1965.0, 112


def measured_peak():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_INT_PEAKS.json")))
        wide = mp["per_sm_per_clk"]["IMAD.WIDE.U32 (carry-chained lo/hi pair, the fr_mul building block)"]
        return wide * SMS * MAX_MHZ * 1e6 / PRODUCTS_PER_MUL / 1e9, \
            f"MEASURED_INT_PEAKS.json: IMAD.WIDE.U32 {wide:.2f}/clk/SM x 148 SM x 1965 MHz / 112 products per Fr mul"
    except (OSError, KeyError, ValueError):
        return 32 * SMS * MAX_MHZ * 1e6 / PRODUCTS_PER_MUL / 1e9, "fallback: IMAD.WIDE half rate (32/clk/SM)"


CHUNK_MAX = 1 << 17    # the library's chunked (cooperative) rounds start at the first round with <= 2^17 elements


def kround_rounds(Dp):
    """Rounds run by k_round launches: k = 2 .. kc - 1, kc = the first round (>= 2) with <= 2^17 elements."""
    k = 2
    while (Dp >> (k - 1)) > CHUNK_MAX:
        k += 1
    return list(range(2, k))

class NvmlClockSampler:
    """SM clock and throttle reasons sampled every 2 ms during the timed region (NVML, in-process)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index, self.samples, self.reasons, self.stop = index, [], set(), False

    def __enter__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def _run(self):
        while not self.stop:
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self.stop = True
        self.t.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "nvml"}


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 100 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def oracle_full_h(D, warm=False):
    """One run of the CPU oracle (streaming C tier, oracle/c zko_tlookup_pair_stream) on workload H at D lookups:
    m, B, every round polynomial and the finals.  Returns (seconds, result, threads)."""
    from oracle import c_oracle as C
    wl = W.activation("H", D=D)
    ch = wl.chal
    chal = C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
    t0 = time.perf_counter()
    res = C.prove_pair_stream(wl.x, wl.y, wl.tx, wl.ty, ch.alpha_f, chal, 0, 2, want_B=False)
    return time.perf_counter() - t0, res, C.num_threads()


def run_reference(args):
    """The oracle (streaming C tier, OpenMP over the host cores) on the full workload H per timed step."""
    world, rank, _ = dist_setup(args.gpus)
    if rank != 0:
        return
    D = 1 << args.log2d
    for _ in range(args.warmup):
        oracle_full_h(1 << 16)          # warm-up: thread pool and caches (a small sample)
    times = []
    for _ in range(args.steps):
        dt, _, cores = oracle_full_h(D)
        times.append(dt)
    t = sum(times) / len(times)
    v = D / t
    sample = f"the full workload H (D=2^{args.log2d} lookups, same generator, SiLU table N=2^16): m, B, every round " \
             f"polynomial, finals; warm-up runs on a 2^16 sample"
    out = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "u32x8 (Fr, exact)", "data": "synthetic",
           "config": {"workload": WORKLOAD, "D": D, "N": 1 << 16, "P": 1, "sample": sample, "same_config": True},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="zkl", choices=["zkl", "reference"])
    ap.add_argument("--log2d", type=int, default=26, help="log2 of the global lookup count (default: H, 2^26)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fs", action="store_true", help="skip the Fiat-Shamir step")
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--inflight", type=int, default=0, help="proofs in flight per rank (default: 2 at P = 1, else 1)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2404_16109_b200 import zkl

    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    D = 1 << args.log2d
    P = world
    Dp = D // P
    wl = W.activation("H", D=D)
    x = torch.from_numpy(wl.x[rank * Dp:(rank + 1) * Dp].copy())
    y = torch.from_numpy(wl.y[rank * Dp:(rank + 1) * Dp].copy())
    tx, ty = torch.from_numpy(wl.tx.copy()), torch.from_numpy(wl.ty.copy())
    N = wl.N
    dev = torch.device("cuda", local)
    # a dedicated (non-default) compute stream: the legacy default stream would serialise with the e2e copy stream
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    nccl_id = None
    if world > 1:
        obj = [zkl.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctx = zkl.Context(local, stream=stream, rank=rank, nranks=world, nccl_id=nccl_id)
    ctx.reserve(Dp, N)
    ch = wl.chal
    chal = zkl.Context.challenges(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
    xd, yd, txd, tyd = (t.to(dev) for t in (x, y, tx, ty))
    T = ctx.vec(N)
    tmem = ctx.table_mem(N)
    m = torch.empty(N, dtype=torch.int32, device=dev)

    use_async = True   # the histogram overlaps the proof; at P > 1 its all-reduce follows it

    def make_step(c, Tv, tm, mv):
        def step(xs, ys, txs, tys):
            # a1 (T) + a2, then a1 (S) fused with a3 (zkl_tlookup_prepare_pair), then a4-a9
            c.import_pair(txs, tys, ch.alpha_f, Tv)
            tab = c.table(Tv, tm)
            c.table_attach_pair(tab, txs, tys, ch.alpha_f)   # pair-range fast path of prepare_pair
            # S stays virtual (only the table keys are kept, S_i = T_key)
            if not use_async:
                c.prepare_pair(xs, ys, ch.alpha_f, D, tab, m=mv, virtual_s=True)
                return c.prove(None, D, tab, mv, chal, args.variant)
            c.set_async(True)
            c.prepare_pair(xs, ys, ch.alpha_f, D, tab, m=mv, virtual_s=True)
            pending = c.prove(None, D, tab, mv, chal, args.variant)
            c.wait()
            c.set_async(False)
            return pending.result()
        return step

    step = make_step(ctx, T, tmem, m)
    # proofs in flight (one rank): lane i = its own context, stream and host thread, taking every other step, so one
    # proof's host-side calls and latency-bound phases overlap the other's rounds (a server keeping requests in
    # flight); each lane's transcript is checked equal to the single-lane one.  At P > 1 one lane (one communicator).
    nlanes = args.inflight if args.inflight else (2 if world == 1 else 1)
    lanes = [(stream, step, ctx)]
    for _ in range(1, nlanes):
        s2 = torch.cuda.Stream(device=dev)
        c2 = zkl.Context(local, stream=s2)
        c2.reserve(Dp, N)
        lanes.append((s2, make_step(c2, c2.vec(N), c2.table_mem(N), torch.empty(N, dtype=torch.int32, device=dev)),
                      c2))

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        pf = step(xd, yd, txd, tyd)
    for ls, lstep, _ in lanes[1:]:
        with torch.cuda.stream(ls):
            for _ in range(args.warmup):
                assert lstep(xd, yd, txd, tyd).evals == pf.evals
    torch.cuda.synchronize(dev)

    def run_timed(nl, steps):
        """steps on nl lanes (steps per lane = steps // nl); device time from the first lane's start event to the
        last lane's end, on the device (the other lanes' streams wait on the start event)."""
        import threading
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        done = [torch.cuda.Event() for _ in range(nl)]
        out = [None] * nl
        e0.record(stream)
        for ls, _, _ in lanes[1:nl]:
            ls.wait_event(e0)

        def run(i):
            ls, lstep, _ = lanes[i]
            with torch.cuda.stream(ls):
                for _ in range(steps // nl):
                    out[i] = lstep(xd, yd, txd, tyd)
                done[i].record(ls)

        th = [threading.Thread(target=run, args=(i,)) for i in range(1, nl)]
        for t in th:
            t.start()
        run(0)
        for t in th:
            t.join()
        for i in range(1, nl):
            stream.wait_event(done[i])
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / ((steps // nl) * nl), out

    # ---------------- timed region: inputs resident in HBM (X, Y int32 512 MiB > L2; S 2 GiB)
    barrier()
    torch.cuda.synchronize(dev)
    l0 = sum(c.launches for _, _, c in lanes)
    with NvmlClockSampler(local) as clk:
        ms, outs = run_timed(nlanes, args.steps * nlanes)
    barrier()
    launches = sum(c.launches for _, _, c in lanes) - l0   # inside the timed region, every lane
    for o in outs:
        assert o.evals == pf.evals and o.finals == pf.finals
    single_ms = ms
    if nlanes > 1:
        single_ms, _ = run_timed(1, args.steps)   # one proof at a time, for the record
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = D / (ms / 1e3)
    # ---------------- per-kernel timing: the same K steps again with CUDA events around every launch (on the
    # launching stream), kept out of the timed region above because recording them costs ~0.4 ms per step
    ctx.set_profiling(True)
    kern, kern_overlap = {}, {}
    for _ in range(args.steps):
        step(xd, yd, txd, tyd)
        for name, kms, _, tag in ctx.profile_read(with_start=True):
            if tag == 0:    # kernels on the critical (ctx) stream; side/aux/low launches overlap it
                kern.setdefault(name, []).append(kms)
            else:
                kern_overlap.setdefault(name, []).append(kms)
    ctx.set_profiling(False)

    # ---------------- Fiat-Shamir mode (f1, single rank): the same step with challenges derived on the device
    fs_ms = None
    if not args.no_fs:   # every P: one all-gather of the round sums per local round at P > 1
        seed = bytes(32)

        fs_async = os.environ.get("ZKL_BENCH_FS_ASYNC", "1") == "1"

        def step_fs():
            ctx.import_pair(txd, tyd, ch.alpha_f, T)
            tab = ctx.table(T, tmem)
            ctx.table_attach_pair(tab, txd, tyd, ch.alpha_f)   # pair-range fast path of prepare_pair
            if not fs_async:
                ctx.prepare_pair(xd, yd, ch.alpha_f, D, tab, m=m, virtual_s=True)
                return ctx.prove_fs(None, D, tab, m, seed, args.variant)
            # as the main step: the histogram on the low-priority stream behind the proof (the table side waits for m)
            ctx.set_async(True)
            ctx.prepare_pair(xd, yd, ch.alpha_f, D, tab, m=m, virtual_s=True)
            pending = ctx.prove_fs(None, D, tab, m, seed, args.variant)
            ctx.wait()
            ctx.set_async(False)
            return pending.result()

        step_fs()
        torch.cuda.synchronize(dev)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            step_fs()
        f1.record(stream)
        torch.cuda.synchronize(dev)
        fs_ms = f0.elapsed_time(f1) / args.steps
        if world > 1:
            t = torch.tensor([fs_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            fs_ms = float(t.item())

    # ---------------- e2e through the library's host-buffer entry point (zkl_tlookup_prove_pair_host): every step
    # copies X, Y, T_X, T_Y from pinned host memory into context-owned device buffers, builds the table, proves and
    # returns the transcript to the host, inside one C call.  On one rank two contexts (two streams, two host threads)
    # take alternate steps, so one step's PCIe copy overlaps the other's proof -- the way a server keeps two requests
    # in flight.  Timed with CUDA events: the first step's start on its stream to the last step's end on its stream.
    xh, yh, txh, tyh = (t.pin_memory() for t in (x, y, tx, ty))
    nctx = int(os.environ.get("ZKL_E2E_INFLIGHT", "0")) or (2 if world == 1 else 1)
    e2e_streams = [torch.cuda.Stream(device=dev) for _ in range(nctx)]
    e2e_ctx = [ctx] if nctx == 1 else []
    for i in range(len(e2e_ctx), nctx):
        c2 = zkl.Context(local, stream=e2e_streams[i], rank=rank, nranks=world)
        c2.reserve(Dp, N)
        e2e_ctx.append(c2)
    if nctx == 1:
        e2e_streams = [stream]
    results = [None] * max(args.steps, 2)

    def e2e_worker(j, n):
        for i in range(j, n, nctx):
            results[i] = e2e_ctx[j].prove_pair_host(xh, yh, txh, tyh, ch.alpha_f, D, chal, args.variant)

    def e2e_run(n):
        import threading as th
        ths = [th.Thread(target=e2e_worker, args=(j, n)) for j in range(nctx)]
        for t_ in ths:
            t_.start()
        for t_ in ths:
            t_.join()

    e2e_run(2)                                   # warm-up (allocates the owned buffers)
    barrier()
    torch.cuda.synchronize(dev)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(e2e_streams[0])
    for st_ in e2e_streams[1:]:
        st_.wait_event(e2)
    e2e_run(args.steps)
    for st_ in e2e_streams[1:]:
        ev = torch.cuda.Event()
        ev.record(st_)
        e2e_streams[0].wait_event(ev)
    e3.record(e2e_streams[0])
    torch.cuda.synchronize(dev)
    ms_e2e = e2.elapsed_time(e3) / args.steps
    if world > 1:
        t = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    for r_ in results[:args.steps]:
        assert r_.evals == pf.evals and r_.finals == pf.finals, "e2e transcript differs from the device-resident step"
    for c2 in e2e_ctx:
        if c2 is not ctx:
            c2.close()
    d = args.log2d
    h2d = 4 * (2 * Dp + 2 * N)
    d2h = 32 * (4 * d + 5)

    # ---------------- roofline of the dominant kernel (largest share of the step) and of the whole step
    peak, peak_basis = measured_peak()
    tot = {}
    for k, v in kern.items():
        k = k.strip("()").split("<")[0] if k.startswith("(") else k
        tot[k] = tot.get(k, 0.0) + sum(v) / args.steps
    dom = max(tot, key=tot.get)
    rounds = kround_rounds(Dp)
    # k_round launches: rounds 2 .. kc-1; round k folds n_old = Dp / 2^(k-2) elements into pairs: 8 muls per new pair
    kr_work = sum(8 * (Dp >> k) for k in rounds)
    # HBM bytes: round 2 reads the 4-byte keys (A, S gathered from the L2-resident table) and writes A', S' (32 B each
    # per new element); rounds > 2 read A, S (64 B per old element) and write A', S' (32 B per old element)
    kr_bytes = sum(36 * Dp if k == 2 else 96 * (Dp >> (k - 2)) for k in rounds)
    work = {"k_round": kr_work, "k_round1_keys": 2 * (Dp // 2)}
    per_step_work = work.get(dom, 0.0)
    achieved = per_step_work / (tot[dom] / 1e3) / 1e9 if per_step_work else None
    traffic, traffic_src = None, None
    try:
        summ = json.load(open(os.path.join(ROOT, "profiles", "r02_ncu_summary.json")))
        if dom in summ and args.log2d == 26 and world == 1:
            traffic = summ[dom]["dram_bytes_per_step"]
            traffic_src = "profiles/r02_ncu_summary.json (ncu dram__bytes_read+write, per step, cold cache)"
    except (OSError, ValueError, KeyError):
        pass
    step_work = 5.0 * D + 16.0 * N                       # algorithmic Fr muls of the whole step (all ranks)
    step_roof_ms = step_work / world / (peak * 1e9) * 1e3
    roofline = {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GFrmul/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "traffic_unit": "bytes per step (all launches of the kernel)", "traffic_source": traffic_src,
                "algorithmic_bytes": kr_bytes if dom == "k_round" else None,
                "work_fr_muls_per_step": per_step_work, "work_rounds": rounds if dom == "k_round" else None,
                "peak_basis": peak_basis, "share_of_step": tot[dom] / single_ms, "kernel_ms_per_step": tot[dom],
                "step": {"fr_muls": step_work, "roofline_ms": step_roof_ms, "frac": step_roof_ms / ms,
                         "basis": "5 Fr muls per lookup (round 1: 2 per pair; rounds >= 2: 8 per new pair) + 16 per "
                                  "table entry, at the measured peak; per rank"}}
    kernels = {k: round(v, 4) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "u32x8 (Fr, exact)", "data": "synthetic",
           "config": {"workload": WORKLOAD, "D": D, "N": N, "P": world, "D_local": Dp, "variant":
                      "paper" if args.variant == 0 else "logup", "parallelism": f"hypercube-top{world}",
                      "schedule": "causal: each round's kernel uses only r_1..r_{k-1}; the small rounds run "
                                  "with a grid barrier per round",
                      "l2": "inputs larger than L2 (X,Y int32 512 MiB; S virtual, keys 256 MiB, folded A,S 2 GiB)",
                      "in_flight": nlanes, "single_proof_ms_per_step": single_ms,
                      "timing": "CUDA events on the device, first lane's start to the last lane's end; ms_per_step = "
                                "that time / steps of all lanes; every lane's transcript checked"},
           "e2e": {"value": D / (ms_e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                   "api": "zkl_tlookup_prove_pair_host (host buffers in, transcript out, one call per step)",
                   "in_flight": nctx},
           "gpu_launches": launches, "roofline": roofline, "clocks": clk.summary(),
           "kernel_ms_per_step": kernels, "kernel_ms_sum": sum(tot.values()),
           "kernel_ms_overlapped": {k: round(sum(v) / args.steps, 4)
                                    for k, v in sorted(kern_overlap.items(), key=lambda kv: -sum(kv[1]))[:8]},
           "fiat_shamir": {"ms_per_step": fs_ms, "lookups_per_s": (D / (fs_ms / 1e3)) if fs_ms else None,
                           "note": "same step, challenges derived on the device (SHA-256 transcript, per-round)"}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dt, res, cores = oracle_full_h(D)
        assert res.evals == pf.evals and res.finals == pf.finals, "the oracle's transcript differs from the GPU's"
        out["cpu_baseline"] = {"value": D / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
                               "sample": f"the full workload H (D=2^{args.log2d}): m, B, every round polynomial, "
                                         f"finals (streaming C tier, {dt:.1f} s); its transcript equals the GPU's",
                               "same_config": True}
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
