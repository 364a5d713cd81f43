"""Benchmark: input triplets/s assembled to CSC on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

A step is one full assembly S = sparse(i, j, s, m, n) of the workload
(default: BASELINE configs[3], the heavy-duplicate random input, m = n = 1e7,
1e8 positions x Poisson(5) repeats, L ~ 5e8 triplets: the largest config
that fits one GPU; --config 1..5 picks another).  Inputs (8 GB) and the
workspace exceed the 126 MB L2, so consecutive steps stream from HBM (no
explicit flush; inputs that fit in L2 are timed step by step after a flush).

Prints ONE JSON line (rank 0):
  value        whole-job triplets/s, device-resident inputs, CUDA events on
               the launching stream, max over ranks
  e2e          the same metric through the public host API
               paper_1406_1066_b200.assemble(numpy arrays in pinned memory)
               -> host CSC (H2D of the triplets and D2H of jc/ir/pr inside)
  roofline     dominant kernel: its algorithmic bytes / its event-timed
               duration vs MEASURED_PEAKS.json hbm_gbs
  path_roofline  compulsory bytes of the whole assembly (16 L + 12 nnz +
               4 (N+1)) / step time
  cpu_baseline the UNMODIFIED reference package (oracle/_ref: stock
               sparseasm.assemble_parallel over its compiled kernels, all
               host threads) on a bounded sample of the same workload (the
               first Ls triplets, ~1 s per run)
  sharded_config_1gpu  (default cfg4 line) cfg5, the sharded config, whole
               on this GPU: the N = 1 point of the multi-GPU runs
Under torchrun with N > 1 ranks: cfg5 split over the ranks (strong scaling),
column-block sharding with one NCCL exchange.
--impl reference runs only that CPU implementation (one sample per step) and
prints its line, with the same `config` as this arm.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input triplets/sec assembled to CSC"
L2_BYTES = 126 << 20
UNIT = "triplets/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """Clock / throttle-reason sampling during the timed region: NVML
    (pynvml: SM clock + throttle reasons, ~1.4 ms per sample, back to back)
    when importable, else nvidia-smi."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, [reason names])
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._bits = (pynvml.nvmlClocksEventReasonHwSlowdown,
                          pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                          pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                          pynvml.nvmlClocksEventReasonSwPowerCap)
            # the max clock does not change: queried once (an NVML query is ~0.7 ms)
            self._max = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        self.samples.append((float(sm), self._max, [n for n, bit in zip(self.NAMES, self._bits) if r & bit]))

    def _sample_smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                  "clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={fields}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        parts = [p.strip() for p in out.stdout.strip().split(",")]
        if len(parts) == 6 and parts[0].replace(".", "").isdigit():
            self.samples.append((float(parts[0]), float(parts[1]),
                                 [n for n, v in zip(self.NAMES, parts[2:]) if v == "Active"]))

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml is not None:
                    self._sample_nvml()
                else:
                    self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.0002 if self._nvml is not None else 0.1)  # NVML: back to back

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(x[0] for x in self.samples),
                "sm_max_mhz": max(x[1] for x in self.samples),
                "reasons": sorted({n for x in self.samples for n in x[2]}),
                "samples": len(self.samples),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


REF_STEP_S = 5.0  # longest timed reference step before the workload is sampled


def reference_sample(ii, jj, s, m, n, target_s=REF_STEP_S):
    """Size the bounded sample of the workload for the reference's CPU path:
    the first Ls triplets (same m, n).  Its run time is fitted as a + b Ls
    from two untimed probe runs (the O((m + n) p) merges of the threaded
    driver are a fixed cost, so a small prefix alone would understate its
    throughput); the whole workload is used when one run fits in
    ``target_s``.  Returns (Ls, req, run, p) with the reference's request
    built once, outside any timing (its run_bench protocol,
    bench.py:146-160)."""
    from oracle import stock

    p = stock.host_threads()
    L = len(ii)

    def timed(k):
        req = stock.request(ii[:k], jj[:k], s[:k], m, n)
        t0 = time.perf_counter()
        stock.parallel(req, p)
        return req, time.perf_counter() - t0

    k0 = min(L, 1 << 22)
    req, t0 = timed(k0)
    Ls = k0
    if k0 < L:
        k1 = min(L, 1 << 24)
        req, t1 = timed(k1)
        Ls = k1
        if k1 < L:
            b_ = max((t1 - t0) / (k1 - k0), 1e-12)
            a_ = max(t1 - b_ * k1, 0.0)
            want = int(min(L, max(k1, (target_s - a_) / b_)))
            if want > k1:
                Ls = want
                req = stock.request(ii[:Ls], jj[:Ls], s[:Ls], m, n)
    return Ls, req, (lambda: stock.parallel(req, p)), p


def cpu_reference_run(ii, jj, s, m, n, budget_s=15.0, max_reps=20):
    """cpu_baseline: the UNMODIFIED reference package (oracle/_ref: its
    threaded driver over its compiled kernels, parallel.py:361-389) with all
    host threads, on a bounded sample of the workload."""
    Ls, req, run, p = reference_sample(ii, jj, s, m, n)
    out = run()  # warm-up (untimed), also the parity reference for the sample
    times = []
    t_start = time.perf_counter()
    while len(times) < max_reps and (time.perf_counter() - t_start) < budget_s:
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    mean = sum(times) / len(times)
    # the reference's serial driver too, one run on a prefix of
    # the sample sized for about 3 s (its throughput is flat in L)
    from oracle import stock

    Lser = min(Ls, 1 << 22)
    rq = stock.request(ii[:Lser], jj[:Lser], s[:Lser], m, n)
    t0 = time.perf_counter()
    stock.serial(rq)
    ts = time.perf_counter() - t0
    if ts < 1.0 and Lser < Ls:
        Lser = int(min(Ls, Lser * max(1.0, 3.0 / max(ts, 1e-3))))
        rq = stock.request(ii[:Lser], jj[:Lser], s[:Lser], m, n)
        t0 = time.perf_counter()
        stock.serial(rq)
        ts = time.perf_counter() - t0
    return dict(kind="reference", cores=p, mean_s=mean, min_s=min(times), reps=len(times), Ls=Ls,
                serial_value=Lser / ts, serial_Ls=Lser), out


def bench_config(w, world: int, shard: bool) -> dict:
    """The workload description both arms print (identical keys): the whole
    job's workload (a sharded run's chunks carry the global name and L)."""
    name = getattr(w, "global_name", w.name)
    L = getattr(w, "global_L", w.L)
    small = 16 * L < L2_BYTES
    return {"workload": name, "L": L, "m": w.m, "n": w.n,
            "l2": ("inputs fit in the 126 MB L2: each step timed alone after a 256 MB flush"
                   if small else
                   "inputs (16 B x L) and workspace exceed the 126 MB L2; no explicit flush"),
            "parallelism": (f"column-block shards over {world} GPUs (contiguous triplet chunk per "
                            "rank, NCCL all-to-all exchange)") if shard else "single"}


def build_workload(cfg: int, device, rank: int, world: int):
    from paper_1406_1066_b200 import workloads as W

    if world > 1 or cfg == 5:
        # BASELINE configs[4], the sharded config: the N = 8000 triangulated
        # mesh (L = 1.152e9), rank r holding a contiguous chunk of its element
        # stream (strong scaling: the whole job is the same at every N)
        Nm = 8000
        cells = Nm * Nm
        c0, c1 = cells * rank // world, cells * (rank + 1) // world
        w = W.fem2d(Nm, device=device, cell_range=(c0, c1))
        w.global_name, w.global_L = f"fem2d_N{Nm}", 18 * cells
        w.name = f"fem2d_N{Nm}_chunk{rank}of{world}"
        return w
    return W.config(cfg, device=device)


def sharded_config_point(w, lib, ctx, asm, dev, stream, steps, warmup):
    """cfg5 (the sharded config) assembled whole on this GPU, device-resident,
    CUDA events on the library's stream: the N = 1 point of the scaling runs
    (which split cfg5 over the ranks)."""
    import torch

    for name in ("ii", "jj", "s"):  # the headline workload's inputs are no longer needed
        setattr(w, name, None)
    torch.cuda.empty_cache()
    w5 = build_workload(5, dev, 0, 1)
    L5, M5, N5 = w5.L, w5.m, w5.n
    jc = torch.empty(N5 + 1, dtype=torch.int32, device=dev)
    ir = torch.empty(L5, dtype=torch.int32, device=dev)
    pr = torch.empty(L5, dtype=torch.float64, device=dev)

    def step():
        rc = lib.sa_assemble_async(ctx, w5.ii.data_ptr(), w5.jj.data_ptr(), w5.s.data_ptr(), 1, L5, M5, N5,
                                   jc.data_ptr(), ir.data_ptr(), pr.data_ptr(), L5)
        if rc:
            raise RuntimeError(asm._msg())

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del w5, jc, ir, pr
    torch.cuda.empty_cache()
    return {"workload": f"fem2d_N8000", "L": L5, "m": M5, "n": N5, "steps": steps,
            "ms_per_step": ms, "value": L5 / (ms * 1e-3), "unit": UNIT}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    # default: configs[3], the largest single-GPU BASELINE config (heavy-duplicate
    # random, L ~ 5e8); under torchrun with N > 1 ranks: configs[4], the
    # sharded config, split over the ranks (its N = 1 point: --config 5)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sharded-point", action="store_true",
                    help="skip the sharded config's one-GPU point (cfg4 runs only)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU (sharded, NCCL) step even with one rank (under torchrun)")
    args = ap.parse_args()
    world, rank, local = _dist()
    if args.warmup < 3:
        args.warmup = 3

    import numpy as np
    import torch

    if args.impl == "reference":
        if rank != 0:
            return
        # the same bits as the GPU arm's workload (generated on the GPU when
        # there is one; input generation is not part of either timed path)
        gen_dev = torch.device("cuda", local) if torch.cuda.is_available() else "cpu"
        # N > 1: the sharded config as the GPU arm runs it, whole (rank 0 holds it)
        w = build_workload(5 if args.gpus > 1 else args.config, gen_dev, 0, 1)
        ii, jj, s = w.ii.cpu().numpy(), w.jj.cpu().numpy(), w.s.cpu().numpy()
        cfg_line, wL = bench_config(w, args.gpus, args.gpus > 1), w.L
        del w.ii, w.jj, w.s  # device copies
        # each step a bounded sample (REF_STEP_S: large enough that the
        # threaded driver's fixed O((m + n) p) merge cost does not understate
        # its throughput); warm-up runs at most 2, and only as many timed
        # steps as fit in about two and a half minutes (at least 3, at most
        # --steps): the line's "steps" is the count actually timed
        Ls, req, run, p = reference_sample(ii, jj, s, w.m, w.n)
        t0 = time.perf_counter()
        run()  # warm-up (also times one step)
        t_step = time.perf_counter() - t0
        for _ in range(min(args.warmup, 2) - 1):
            run()
        nsteps = int(min(args.steps, max(3, 150.0 // max(t_step, 1e-3))))
        times = []
        for _ in range(nsteps):
            t0 = time.perf_counter()
            run()
            times.append(time.perf_counter() - t0)
        mean = sum(times) / len(times)
        val = Ls / mean
        sample = (f"first {Ls} of the workload's {wL} triplets (same m, n) per step, "
                  f"stock sparseasm.assemble_parallel(req, p={p}) from oracle/_ref")
        line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
                "steps": nsteps, "steps_requested": args.steps, "warmup": args.warmup,
                "ms_per_step": mean * 1e3,
                "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": cfg_line,
                "cpu_baseline": {"value": val, "unit": UNIT, "cores": p, "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import paper_1406_1066_b200 as sa
    from paper_1406_1066_b200 import _capi

    shard = world > 1 or args.sharded

    if shard:
        import torch.distributed as dist

        # communicator set-up lines (nranks, transport) on stderr for the record
        # (the image's NCCL_DEBUG=VERSION prints only the banner)
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() in ("", "VERSION", "WARN"):
            os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")

        # stdout carries only the JSON line: the communicator is created (and
        # NCCL prints its version banner, NCCL_DEBUG=VERSION in this image)
        # with fd 1 pointing at stderr
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w = build_workload(args.config, dev, rank, world)
    torch.cuda.synchronize()
    L, M, N = w.L, w.m, w.n
    asm = sa.default_assembler(local)
    lib, ctx = asm.lib, asm.ctx
    cap = L
    jc = torch.empty(N + 1, dtype=torch.int32, device=dev)
    ir = torch.empty(cap, dtype=torch.int32, device=dev)
    pr = torch.empty(cap, dtype=torch.float64, device=dev)
    asm._bind_stream()
    stream = torch.cuda.current_stream(dev)

    if shard:
        # column-block sharding: histogram + all_reduce, stable partition,
        # NCCL all_to_all of the triplets, local CUDA assembly, nnz all_gather
        from paper_1406_1066_b200.distributed import assemble_sharded, gpu_local_assembler

        local_asm = gpu_local_assembler(local)
        shard_info = {}
        shard_out = {}  # result buffers reused across steps (as the single-GPU step's jc / ir / pr)

        def step():
            res = assemble_sharded(w.ii, w.jj, w.s, M, N, local_asm, out=shard_out)
            shard_info["nnz"] = res.nnz_total
            shard_info["nnz_local"] = int(res.ir.numel())
            shard_info["n_local"] = res.col_hi - res.col_lo
            shard_info["launches"] = res.launches
            shard_info["sent_remote"] = res.sent_remote
            shard_info["recv"] = res.recv_triplets
    else:
        def step():
            rc = lib.sa_assemble_async(ctx, w.ii.data_ptr(), w.jj.data_ptr(), w.s.data_ptr(), 1, L,
                                       M, N, jc.data_ptr(), ir.data_ptr(), pr.data_ptr(), cap)
            if rc:
                raise RuntimeError(asm._msg())

    # correctness of the configuration (device result must be complete)
    step()
    import ctypes

    if shard:
        nnz = shard_info["nnz"]
        launches_per_step = shard_info["launches"]  # partition + local assembly
    else:
        nnz_c = ctypes.c_int64(0)
        rc = lib.sa_finish(ctx, ctypes.byref(nnz_c), None, None)
        if rc:
            raise RuntimeError(f"assembly failed: {asm._msg()}")
        nnz = nnz_c.value
        launches_per_step = lib.sa_last_launch_count(ctx)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if shard:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # inputs that fit in the 126 MB L2 (cfg1): every step timed on its own,
    # the L2 flushed between steps (a 256 MB write outside the timed events)
    small = 16 * L < L2_BYTES
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if small else None
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if small:
            tot = 0.0
            for _ in range(args.steps):
                flush.zero_()
                ev0.record(stream)
                step()
                ev1.record(stream)
                ev1.synchronize()
                tot += ev0.elapsed_time(ev1)
            ms = tot / args.steps
        else:
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1) / args.steps
    if shard:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()

    # per-kernel breakdown (events inside the library on the same stream)
    lib.sa_enable_timing(ctx, 1)
    kt = {}
    nk = 0
    reps = max(3, min(args.steps, 10))
    for _ in range(reps):
        step()
        arr = (ctypes.c_float * 16)()
        names = (ctypes.c_char_p * 16)()
        nk = lib.sa_last_kernel_times(ctx, 16, arr, names)
        for k in range(nk):
            kt.setdefault(names[k].decode(), []).append(arr[k])
    lib.sa_enable_timing(ctx, 0)
    kern_ms = {k: sum(v) / len(v) for k, v in kt.items()}
    dom = max(kern_ms, key=kern_ms.get)
    # algorithmic bytes per launch of each kernel ("kernels"); at
    # N > 1 the rank's own assembly: its chunk, its column block, its nnz
    # (received triplets are few for the element-ordered meshes)
    nl = shard_info["nnz_local"] if shard else nnz
    Nl = shard_info["n_local"] if shard else N
    Lv = L  # valid triplets (every index is valid in the BASELINE workloads)
    alg = {
        # column-cursor pipeline (sa_kernels.cu, sa_tile.cu)
        "k_init": 4 * (Nl + 1),
        "k_colcount": 4 * L,
        "k_col_scan": 8 * Nl,
        "k_scatter": 16 * L,
        "k_bigcol": 0,
        "k_tile_fold": 16 * L + 8 * Nl + 12 * nl + 4 * (Nl + 1),
        # column-block radix path (sa_radix.cu): per pass an upsweep over the
        # columns and a 16 B in / 16 B out partition; the fold reads every
        # partitioned triplet once and writes the CSC
        "k_rup0": 4 * L, "k_rup1": 4 * Lv, "k_rup2": 4 * Lv,
        "k_rpass0": 32 * Lv, "k_rpass1": 32 * Lv, "k_rpass2": 32 * Lv,
        "k_rbounds": 0, "k_rbig": 0,
        "k_rfold": 16 * Lv + 12 * nl + 4 * (Nl + 1),
    }
    peak_gbs, peak_kind = _peaks()
    dom_gbs = alg.get(dom, 0) / (kern_ms[dom] * 1e-3) / 1e9
    # whole job: every rank's triplets read, the global CSC written, over
    # world x the per-GPU peak
    compulsory = 16 * getattr(w, "global_L", L * world) + 12 * nnz + 4 * (N + 1)
    path_gbs = compulsory / (ms * 1e-3) / 1e9 / world
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(tpath):
        try:
            rec = json.load(open(tpath)).get(w.name, {}).get(dom)
            if rec:
                traffic = rec["dram_read_bytes"] + rec["dram_write_bytes"]
        except Exception:
            traffic = None

    # end-to-end through the public host API (pinned host inputs)
    hi = torch.empty(L, dtype=torch.int32, pin_memory=True)
    hj = torch.empty(L, dtype=torch.int32, pin_memory=True)
    hs = torch.empty(L, dtype=torch.float64, pin_memory=True)
    hi.copy_(w.ii)
    hj.copy_(w.jj)
    hs.copy_(w.s)
    hin, hjn, hsn = hi.numpy(), hj.numpy(), hs.numpy()
    d2h = 4 * (N + 1) + 12 * nnz
    if shard:
        # host chunk -> device, sharded assembly, the rank's column block -> host
        pinned = {}

        def to_pinned(name, x):  # page-locked result buffers, reused across calls
            buf = pinned.get(name)
            if buf is None or buf.numel() < x.numel():
                buf = pinned[name] = torch.empty(int(x.numel() * 1.25) + 16, dtype=x.dtype,
                                                 pin_memory=True)
            out_ = buf[: x.numel()]
            out_.copy_(x, non_blocking=True)
            return out_

        def e2e_call():
            di = hi.to(dev, non_blocking=True)
            dj = hj.to(dev, non_blocking=True)
            ds = hs.to(dev, non_blocking=True)
            res = assemble_sharded(di, dj, ds, M, N, local_asm, out=shard_out)
            outs = (to_pinned("jc", res.jc), to_pinned("ir", res.ir), to_pinned("pr", res.pr))
            torch.cuda.current_stream(dev).synchronize()
            return outs

        for _ in range(2):  # warm-up (allocator, page-locked buffers)
            jc_h, ir_h, pr_h = e2e_call()
        d2h = 8 * len(jc_h) + 12 * len(ir_h)
        out = None
    else:
        def e2e_call():
            return sa.assemble(hin, hjn, hsn, m=M, n=N, device=local)

        for _ in range(3):  # warm-up (fills the page-locked output cache for alternating results)
            out = e2e_call()
    e2e_t = []
    for _ in range(max(1, args.e2e_steps)):
        torch.cuda.synchronize()
        if shard:
            dist.barrier()
        t0 = time.perf_counter()
        r = e2e_call()
        e2e_t.append(time.perf_counter() - t0)
        if not shard:
            out = r
    e2e_s = sum(e2e_t) / len(e2e_t)
    if shard:
        t = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    cpu = None
    parity = None
    if rank == 0 and not shard and not args.no_cpu_baseline:
        info, ref = cpu_reference_run(hin, hjn, hsn, M, N)
        Ls = info["Ls"]
        # parity on the sample: the public API on the same Ls triplets
        mine = out if Ls == L else sa.assemble(hin[:Ls], hjn[:Ls], hsn[:Ls], m=M, n=N, device=local)
        parity = bool(mine.same_as(ref))
        cpu = {"value": Ls / info["mean_s"], "unit": UNIT, "cores": info["cores"], "kind": info["kind"],
               "serial": {"value": info["serial_value"], "unit": UNIT, "cores": 1,
                          "sample": f"first {info['serial_Ls']} triplets, stock sparseasm.assemble_serial"},
               "sample": f"first {Ls} of {L} triplets (same m, n), stock sparseasm.assemble_parallel "
                         f"(oracle/_ref) on {info['cores']} threads, {info['reps']} timed runs after "
                         f"1 warm-up, mean {info['mean_s'] * 1e3:.1f} ms"}

    # the sharded config's one-GPU point (the N > 1 runs split it over the
    # ranks): measured here too, so a scaling curve has its N = 1 reference
    sharded_1gpu = None
    cfg_line = bench_config(w, world, shard)
    if rank == 0 and not shard and args.config == 4 and not args.no_sharded_point:
        sharded_1gpu = sharded_config_point(w, lib, ctx, asm, dev, stream, max(3, min(args.steps, 10)),
                                            args.warmup)

    if rank != 0:
        if shard:
            dist.destroy_process_group()
        return
    Ltot = getattr(w, "global_L", L) if shard else L  # every rank's triplets
    value = Ltot / (ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if shard else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg_line,
        "nnz": nnz,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": dom_gbs, "peak": peak_gbs,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": dom_gbs / peak_gbs,
                     "traffic": traffic, "alg_bytes_per_launch": alg.get(dom),
                     "launch_ms": kern_ms[dom]},
        "path_roofline": {"compulsory_bytes": compulsory, "achieved": path_gbs, "peak": peak_gbs,
                          "unit": "GB/s", "frac": path_gbs / peak_gbs},
        "kernel_ms": kern_ms,
        "e2e": {"value": (getattr(w, "global_L", L * world) if shard else L) / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 16 * L,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3},
        "gpu_launches": launches_per_step * args.steps,
        "launches_per_step": launches_per_step,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "parity_vs_cpu_reference": parity,
    }
    if sharded_1gpu is not None:
        line["sharded_config_1gpu"] = sharded_1gpu
    if shard:
        line["exchange"] = {"sent_remote_triplets_rank0": shard_info.get("sent_remote"),
                            "received_triplets_rank0": shard_info.get("recv"),
                            "collectives": "all_reduce(block histogram), all_to_all(triplets), "
                                           "all_gather(nnz) over NCCL"}
    print(json.dumps(line), flush=True)
    if shard:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
