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

`--impl reference` times the CPU oracle (oracle/c, the C tier, as it stands) on a bounded sample of the
same workload on the host cores (rank 0 only).
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
# ALU roofline: 148 SMs x 64 IMAD lanes/clk x 1965 MHz; one 8x32-bit Montgomery Fr mul needs
# 120 32x32->64 products (64 operand + 56 reduction, r0 = 1), each 2 lane-slots (IMAD.WIDE is half rate).
SMS, IMAD_PER_CLK, MAX_MHZ, SLOTS_PER_MUL = 148, 64, 1965.0, 240
PEAK_GFRMUL = SMS * IMAD_PER_CLK * MAX_MHZ * 1e6 / SLOTS_PER_MUL / 1e9

# Algorithmic Fr multiplications per launch of each kernel, as a function of the
# element count the launch covers (n_old for the fold rounds, D_local for the inversion passes).
def kernel_work(name: str, n: int) -> float:
    if name == "k_inv_fwd":
        return 1.0 * n                      # prefix products
    if name == "k_inv_bwd":
        return 3.0 * n                      # 2 backward + round-1 (dA dS) * E_lo per pair
    if name.startswith("k_round"):
        return 2.0 * n                      # per new pair: 4 fold + 4 eval = 8 muls per 4 old elements
    if name == "k_import_pair_dev":
        return 2.0 * n
    return 0.0


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


def run_reference(args):
    """The oracle (C tier, OpenMP over the host cores) on a bounded sample of H per step."""
    world, rank, _ = dist_setup(args.gpus)
    if rank != 0:
        return
    from oracle import c_oracle as C
    from oracle import tlookup as TL
    Ds = 1 << args.ref_log2
    wl = W.activation("H", D=Ds)
    S, T = C.inputs_from_workload(wl)
    ch = TL.challenges_from(wl.chal)
    chal = C.chal_array(ch.beta, ch.alpha1, ch.alpha2, ch.u, ch.r)
    for _ in range(args.warmup):
        C.prove(S, T, chal, 0, want_A=False, want_B=False)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        C.prove(S, T, chal, 0, want_A=False, want_B=False)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    v = Ds / t
    sample = f"D=2^{args.ref_log2} lookups of workload H (same generator, SiLU table N=2^16), full m, A, B, transcript"
    cores = C.num_threads()
    out = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "u32x8 (Fr, exact)", "data": "synthetic",
           "config": {"workload": WORKLOAD, "D": 1 << 26, "N": 1 << 16, "P": 1, "sample_D": Ds, "sample": sample},
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
    ap.add_argument("--ref-log2", type=int, default=21, help="oracle sample size (cpu_baseline / reference arm)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--variant", type=int, default=0)
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

    use_async = world == 1   # async mode is single-rank: the histogram overlaps the proof

    def step(xs, ys, txs, tys):
        # a1 (T) + a2, then a1 (S) fused with a3 (zkl_tlookup_prepare_pair), then a4-a9
        ctx.import_pair(txs, tys, ch.alpha_f, T)
        tab = ctx.table(T, tmem)
        ctx.table_attach_pair(tab, txs, tys, ch.alpha_f)   # pair-range fast path of prepare_pair
        # S stays virtual (only the table keys are kept, S_i = T_key)
        if not use_async:
            ctx.prepare_pair(xs, ys, ch.alpha_f, D, tab, m=m, virtual_s=True)
            return ctx.prove(None, D, tab, m, chal, args.variant)
        ctx.set_async(True)
        ctx.prepare_pair(xs, ys, ch.alpha_f, D, tab, m=m, virtual_s=True)
        pending = ctx.prove(None, D, tab, m, chal, args.variant)
        ctx.wait()
        ctx.set_async(False)
        return pending.result()

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        pf = step(xd, yd, txd, tyd)
    # ---------------- timed region: inputs resident in HBM (X, Y int32 512 MiB > L2; S 2 GiB)
    barrier()
    torch.cuda.synchronize(dev)
    l0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with NvmlClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            pf = step(xd, yd, txd, tyd)
        e1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    launches = ctx.launches - l0
    ms = e0.elapsed_time(e1) / args.steps
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
    if world == 1:
        seed = bytes(32)

        def step_fs():
            ctx.import_pair(txd, tyd, ch.alpha_f, T)
            tab = ctx.table(T, tmem)
            ctx.table_attach_pair(tab, txd, tyd, ch.alpha_f)   # pair-range fast path of prepare_pair
            ctx.prepare_pair(xd, yd, ch.alpha_f, D, tab, m=m, virtual_s=True)   # synchronous: a background
            return ctx.prove_fs(None, D, tab, m, seed, args.variant)   # histogram only slows the FS rounds

        step_fs()
        torch.cuda.synchronize(dev)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            step_fs()
        f1.record(stream)
        torch.cuda.synchronize(dev)
        fs_ms = f0.elapsed_time(f1) / args.steps

    # ---------------- e2e: host (pinned) X, Y, T_X, T_Y -> device each step, transcript back to the host.
    # Double-buffered: step i+1's inputs are copied on a copy stream while step i computes, so every step's
    # H2D copy and D2H transcript read are inside the timed region and the PCIe transfer overlaps the proof.
    xh, yh, txh, tyh = (t.pin_memory() for t in (x, y, tx, ty))
    bufs = [tuple(torch.empty_like(t) for t in (xd, yd, txd, tyd)) for _ in range(2)]
    cstream = torch.cuda.Stream(device=dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]

    def issue_copy(i):
        b = bufs[i % 2]
        with torch.cuda.stream(cstream):
            for dst, src in zip(b, (xh, yh, txh, tyh)):
                dst.copy_(src, non_blocking=True)
            copied[i % 2].record(cstream)

    def e2e_steps(n):
        issue_copy(0)
        res = None
        for i in range(n):
            if i + 1 < n:
                issue_copy(i + 1)          # the other buffer: its previous step (i - 1) has completed
            stream.wait_event(copied[i % 2])
            res = step(*bufs[i % 2])       # returns after the transcript is on the host
        return res

    e2e_steps(2)
    barrier()
    torch.cuda.synchronize(dev)
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    pe = e2e_steps(args.steps)
    e3.record(stream)
    torch.cuda.synchronize(dev)
    ms_e2e = e2.elapsed_time(e3) / args.steps
    if world > 1:
        t = torch.tensor([ms_e2e], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    assert pe.evals == pf.evals and pe.finals == pf.finals, "e2e transcript differs"
    d = args.log2d
    h2d = 4 * (2 * Dp + 2 * N)
    d2h = 32 * (4 * d + 5)

    # ---------------- roofline of the dominant kernel (largest share of the step)
    tot = {}
    for k, v in kern.items():
        k = k.strip("()").split("<")[0] if k.startswith("(") else k
        tot[k] = tot.get(k, 0.0) + sum(v) / args.steps
    dom = max(tot, key=tot.get)
    per_step_work = 0.0
    if dom == "k_inv_fwd" or dom == "k_inv_bwd":
        per_step_work = kernel_work(dom, Dp)
    elif dom.startswith("k_round"):
        n_old = Dp
        while n_old > 4096:                   # rounds 2.. fold from n_old = Dp, Dp/2, ...
            per_step_work += kernel_work(dom, n_old)
            n_old //= 2
    elif dom in ("k_import_pair_dev", "k_import_pair_index"):
        per_step_work = kernel_work("k_import_pair_dev", Dp)
    achieved = per_step_work / (tot[dom] / 1e3) / 1e9 if per_step_work else None
    # DRAM traffic of the dominant kernel per step, from the committed ncu capture of the same workload
    # (profiles/r01_ncu_summary.json: dram__bytes_read.sum + dram__bytes_write.sum over its launches)
    traffic, traffic_src = None, None
    try:
        summ = json.load(open(os.path.join(ROOT, "profiles", "r01_ncu_summary.json")))
        if dom in summ and args.log2d == 26 and world == 1:
            traffic = summ[dom]["dram_bytes_per_step"]
            traffic_src = "profiles/r01_ncu_summary.json (ncu dram__bytes_read+write, per step, cold cache)"
    except (OSError, ValueError, KeyError):
        pass
    # algorithmic bytes per step of the dominant kernel: fold rounds read 64 B and write 32 B per new pair-half
    alg_bytes = None
    if dom == "k_round":
        alg_bytes, n_old = 0, Dp
        while n_old > 4096:
            alg_bytes += 2 * 32 * n_old + 2 * 32 * n_old // 2
            n_old //= 2
    step_ms_sum = sum(tot.values())
    roofline = {"bound": "alu", "kernel": dom, "achieved": achieved, "peak": PEAK_GFRMUL, "unit": "GFrmul/s",
                "frac": (achieved / PEAK_GFRMUL) if achieved else None, "traffic": traffic,
                "traffic_unit": "bytes per step (all launches of the kernel)", "traffic_source": traffic_src,
                "algorithmic_bytes": alg_bytes, "work_fr_muls_per_step": per_step_work,
                "peak_basis": "148 SM x 64 IMAD lanes/clk x 1965 MHz / 240 lane-slots per 8x32 Montgomery Fr mul",
                "share_of_step": tot[dom] / ms, "kernel_ms_per_step": tot[dom]}
    # whole-proof work-based fraction (all kernels): Fr muls of the algorithm per lookup / time
    kernels = {k: round(v, 4) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])}

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "u32x8 (Fr, exact)", "data": "synthetic",
           "config": {"workload": WORKLOAD, "D": D, "N": N, "P": world, "D_local": Dp, "variant":
                      "paper" if args.variant == 0 else "logup", "parallelism": f"hypercube-top{world}",
                      "l2": "inputs larger than L2 (X,Y int32 512 MiB; S virtual, keys 256 MiB, folded A,S 2 GiB)"},
           "e2e": {"value": D / (ms_e2e / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
           "gpu_launches": launches, "roofline": roofline, "clocks": clk.summary(),
           "kernel_ms_per_step": kernels, "kernel_ms_sum": step_ms_sum,
           "kernel_ms_overlapped": {k: round(sum(v) / args.steps, 4)
                                    for k, v in sorted(kern_overlap.items(), key=lambda kv: -sum(kv[1]))[:8]},
           "fiat_shamir": {"ms_per_step": fs_ms, "lookups_per_s": (D / (fs_ms / 1e3)) if fs_ms else None,
                           "note": "same step, challenges derived on the device (SHA-256 transcript, per-round)"}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import c_oracle as C
        from oracle import tlookup as TL
        Ds = 1 << args.ref_log2
        wls = W.activation("H", D=Ds)
        Sc, Tc = C.inputs_from_workload(wls)
        chs = TL.challenges_from(wls.chal)
        t0 = time.perf_counter()
        C.prove(Sc, Tc, C.chal_array(chs.beta, chs.alpha1, chs.alpha2, chs.u, chs.r), 0, want_A=False,
                want_B=False)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": Ds / dt, "unit": UNIT, "cores": C.num_threads(), "kind": "oracle",
                               "sample": f"D=2^{args.ref_log2} lookups of workload H, full m, A, B, transcript "
                                         f"(C tier, {dt:.1f} s)"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
