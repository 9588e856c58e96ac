"""Benchmark of the maximum-path call (BASELINE.json metric: MAS Gcells/s
(B*T*S / time) and ms/batch at B32 T1024 S8192 vs the CPU reference).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c5]

One step = the whole maximum-path call on one batch of config 3
(B=32 items per GPU, T=1024, S=8192, fp32 log-likelihoods from the
reference's own generator bench::generate_random_batch, generated
bit-identically on the device): K1 forward (direction bits + fused NonFinite
check + fused zero fill of the uint8 [B,T,S] output) and K2 backtrack (the
ones of the alignment), with inputs resident in HBM.  Inputs (1.07 GB per
GPU) are larger than L2 (126 MB), so no flush is needed between steps.

Under torchrun each rank aligns its own 32-item shard (items [32r, 32r+32)
of generate_random_batch(32 N, ...)): weak scaling, no collective on the data
path; NCCL is used only for the start/stop barrier and the max-over-ranks
timing.  `--config c5` is BASELINE's batch-sharded sweep instead: the fixed
batch generate_random_batch(256, 512, 4096, 0) split over the N ranks by
shard.shard_ranges (strong scaling).  `--gpus N` without torchrun's
environment re-launches this script under torch.distributed.run with N ranks
(127.0.0.1 rendezvous).

`--impl reference` times the reference's own CPU engine (oracle/_ref, the
unmodified /root/reference/proj/src compiled in place) on this box's host
cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_CELL = 4 + 1 / 8 + 1  # q read + direction bit + uint8 output
METRIC = "MAS Gcells/s (B*T*S/time) and ms/batch at B32 T1024 S8192 vs CPU ref"
# BASELINE.json configs: c3 (the metric's config, 32 items per GPU, weak
# scaling) and c5 (256 items split over the GPUs, strong scaling).
CONFIGS = {
    "c3": {"B": 32, "T": 1024, "S": 8192, "scaling": "weak",
           "workload": "c3: B32 T1024 S8192 fp32 maximum-path (align -> uint8 [B,T,S]), per GPU"},
    "c5": {"B": 256, "T": 512, "S": 4096, "scaling": "strong",
           "workload": "c5: B256 T512 S4096 fp32 maximum-path (align -> uint8 [B,T,S]), "
                       "batch-sharded over the GPUs"},
}
L2_NOTE = "inputs larger than L2 (q per GPU >= 134 MB vs 126 MB L2), no flush"


def workload_config(name, world):
    """The `config` object both arms print (workload keys only, so the
    driver's same_config check compares like with like)."""
    c = CONFIGS[name]
    B = c["B"] * world if c["scaling"] == "weak" else c["B"]
    return {"workload": c["workload"], "B": c["B"], "T": c["T"], "S": c["S"],
            "global_batch": B, "l2": L2_NOTE}


def rank_items(name, rank, world):
    """[b0, b1) of the batch this rank aligns."""
    c = CONFIGS[name]
    if c["scaling"] == "weak":
        return rank * c["B"], (rank + 1) * c["B"]
    from paper_2409_07704_b200.shard import shard_ranges

    return shard_ranges(c["B"], world)[rank]


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _bf16_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"])
    except Exception:
        return 2250.0  # B200 dense bf16 nominal


def _ncu_traffic():
    """dram bytes per launch of the forward kernel from the committed
    `ncu --set full` summary (profiles/ncu_fwd_latest.json), if present."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_fwd_latest.json")) as f:
            d = json.load(f)
        if d.get("workload") == "c3":
            return float(d["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


class ClockSampler:
    """NVML SM clock + throttle reasons sampled in a thread during the timed
    region (the recipe's nvidia-smi clocks line, at a finer period)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index, period=0.002):
        self.samples, self.reasons = [], 0
        self.period = period
        self.ok = False
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(self.period)

    def sample(self):
        if not self.ok:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
        except Exception:
            pass

    def __enter__(self):
        self.sample()
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.th.join()
        self.sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples),
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b
                            and n != "gpu_idle"]}


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_reference_leg(steps, warmup, budget_s=None, config="c3"):
    """Times monoalign::align (parallel engine, threads=0 = all host threads,
    capped at B by the engine, parallel.cpp:86-91) on a pre-built batch of
    the config (c3: 32 items; c5: the 256-item batch).  Returns (ms list,
    cores, sample description, cells per call)."""
    from oracle.oracle import Reference, build

    c = CONFIGS[config]
    build()
    ref = Reference()
    hw = ref.hardware_threads()
    batch = ref.timed_batch(c["B"], c["T"], c["S"], 0)
    try:
        for _ in range(warmup):
            batch.time("parallel", 0)
        ms = []
        t0 = time.perf_counter()
        while True:
            ms.append(batch.time("parallel", 0))
            if budget_s is None and len(ms) >= steps:
                break
            if budget_s is not None and (time.perf_counter() - t0 >= budget_s or len(ms) >= steps):
                break
    finally:
        batch.close()
    cores = min(hw, c["B"])
    sample = (f"full {config} batch ({c['B']}x{c['T']}x{c['S']}) per align call, {len(ms)} "
              f"call(s), monoalign::align parallel engine, threads=0 -> {cores} workers of {hw} "
              f"hardware threads, timed with steady_clock around align only")
    return ms, cores, sample, c["B"] * c["T"] * c["S"]


def run_reference(args):
    rank, world, _ = _dist()
    if rank != 0:
        return 0
    ms, cores, sample, cells = cpu_reference_leg(args.steps, args.warmup, config=args.config)
    tot = sum(ms) / 1e3
    value = cells * len(ms) / tot / 1e9
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "Gcells/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": len(ms), "warmup": args.warmup,
        "ms_per_step": round(statistics.mean(ms), 3), "higher_is_better": True,
        "scaling": CONFIGS[args.config]["scaling"], "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(args.config, world),
        "parallelism": "host threads",
        "cpu_baseline": {"value": round(value, 4), "unit": "Gcells/s", "cores": cores,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "Gcells/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2409_07704_b200 as mas
    from paper_2409_07704_b200 import _lib

    rank, world, local = _dist()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    c = CONFIGS[args.config]
    b0, b1 = rank_items(args.config, rank, world)
    B, T, S = b1 - b0, c["T"], c["S"]
    cells = B * T * S
    total_cells = (c["B"] * world if c["scaling"] == "weak" else c["B"]) * T * S

    # Inputs: this rank's shard [b0, b1) of generate_random_batch(., T, S, 0).
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        q = mas.generate_device(B, T, S, 0, first_item=b0, device=dev)
        out = torch.empty((B, T, S), dtype=torch.uint8, device=dev)
    plan = mas.Plan(B, T, S)
    geom = plan.geometry
    FWD, BT = _lib.MAS_PART_FORWARD, _lib.MAS_PART_BACKTRACK

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            plan.enqueue(q, out, stream=stream)
        plan.finish(q, stream=stream)  # no NonFinite / validation error

    K = args.steps
    # (1) Per-kernel durations and the single-batch latency: K1 and K2 of each
    # step bracketed by events (untimed for the headline).
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    torch.cuda.synchronize(dev)
    for k in range(K):
        ev[k][0].record(stream)
        plan.enqueue(q, out, stream=stream, parts=FWD)
        ev[k][1].record(stream)
        plan.enqueue(q, out, stream=stream, parts=BT)
        ev[k][2].record(stream)
    torch.cuda.synchronize(dev)
    plan.finish(q, stream=stream)
    fwd_ms = [e[0].elapsed_time(e[1]) for e in ev]
    bt_ms = [e[1].elapsed_time(e[2]) for e in ev]
    # the single-batch latency as a caller sees it: one whole enqueue (K1,
    # then K2 launched early and waiting on K1 through programmatic dependent
    # launch) between two events -- the split above delays K2's launch
    lat = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    for k in range(K):
        lat[k][0].record(stream)
        plan.enqueue(q, out, stream=stream)
        lat[k][1].record(stream)
        torch.cuda.synchronize(dev)
    plan.finish(q, stream=stream)
    latency_ms = statistics.median(e[0].elapsed_time(e[1]) for e in lat)
    # Sanity (outside the timed region): exactly one 1 per column of every item.
    col = out.sum(dim=1, dtype=torch.int32)
    assert bool((col == 1).all()), "alignment invariant violated"

    # (2) The headline: K batches back to back through a pipelined plan --
    # batch k's backtrack runs alongside batch k+1's forward (programmatic
    # dependent launch, two direction-word buffers), each batch writing its
    # own output buffer (two, alternating).
    pplan = mas.Plan(B, T, S, pipelined=True)
    outs = [out, torch.empty_like(out)]
    with torch.cuda.stream(stream):
        for k in range(max(args.warmup, 3)):
            pplan.enqueue(q, outs[k % 2], stream=stream)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    with clocks:
        t_start.record(stream)
        for k in range(K):
            pplan.enqueue(q, outs[k % 2], stream=stream)
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    pplan.finish(q, stream=stream)
    launches_per_step = 2  # mas_fwd4 + bt_walk
    elapsed_ms = t_start.elapsed_time(t_end)
    assert torch.equal(outs[0], outs[1]), "pipelined batches differ"
    assert bool((outs[1].sum(dim=1, dtype=torch.int32) == 1).all()), "pipelined invariant"
    del pplan

    tmax = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    elapsed_ms = float(tmax.item())
    value = total_cells * K / (elapsed_ms / 1e3) / 1e9

    # ---- e2e: the C-ABI host entry point with pinned HOST buffers ----------
    lib = _lib.load()
    hq = torch.empty((B, T, S), dtype=torch.float32, pin_memory=True)
    hq.copy_(q)
    hout = torch.empty((B, T, S), dtype=torch.uint8, pin_memory=True)
    cfg = mas.api._make_config("parallel", -1e32, 0)
    err = _lib.MasError()

    def host_call():
        rc = lib.mas_align_host(hq.data_ptr(), B, T, S, None, ctypes.byref(cfg),
                                hout.data_ptr(), None, ctypes.byref(err))
        _lib.raise_for(rc, err)

    e2e_steps = max(3, min(K, 10))
    for _ in range(2):
        host_call()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        host_call()
    torch.cuda.synchronize(dev)
    e2e_s = torch.tensor([time.perf_counter() - t0], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = total_cells * e2e_steps / float(e2e_s.item()) / 1e9
    assert torch.equal(hout, out.cpu()), "host entry point differs from the device path"
    h2d = B * T * S * 4
    d2h = B * T * S + 4 * B  # alignment bytes + NonFinite flags
    # the e2e roofline: a plain pinned host -> device copy of the same input
    # bytes on this box (the host path is bound by that link)
    dq = torch.empty_like(q)
    dq.copy_(hq, non_blocking=True)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(3):
        dq.copy_(hq, non_blocking=True)
    torch.cuda.synchronize(dev)
    h2d_gbs = 3 * h2d / (time.perf_counter() - t0) / 1e9
    del dq

    # ---- secondary: durations only, no dense output
    dur = torch.empty((B, T), dtype=torch.int32, device=dev)
    with torch.cuda.stream(stream):
        for _ in range(3):
            plan.enqueue(q, stream=stream, durations=dur)
    torch.cuda.synchronize(dev)
    d0 = torch.cuda.Event(enable_timing=True)
    d1 = torch.cuda.Event(enable_timing=True)
    d0.record(stream)
    for _ in range(K):
        plan.enqueue(q, stream=stream, durations=dur)
    d1.record(stream)
    torch.cuda.synchronize(dev)
    dur_ms = d0.elapsed_time(d1) / K
    assert torch.equal(dur, out.sum(dim=2, dtype=torch.int32)), "durations != alignment row sums"
    hdur = torch.empty((B, T), dtype=torch.int32, pin_memory=True)

    def host_dur_call():
        rc = lib.mas_align_host_ex(hq.data_ptr(), B, T, S, None, ctypes.byref(cfg), None, None,
                                   hdur.data_ptr(), ctypes.byref(err))
        _lib.raise_for(rc, err)

    host_dur_call()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        host_dur_call()
    e2e_dur_s = time.perf_counter() - t0
    # ---- the reference binding's own path: numpy (pageable) in, numpy out
    import numpy as np

    q_np = np.array(hq.numpy(), copy=True)  # pageable, like monoalign.align(values)
    for _ in range(2):  # steady state: the pinned output blocks are cached after two calls
        out_np = mas.align(q_np)
    t0 = time.perf_counter()
    np_steps = 3
    for _ in range(np_steps):
        out_np = mas.align(q_np)
    np_s = (time.perf_counter() - t0) / np_steps
    assert np.array_equal(out_np, hout.numpy()), "numpy path differs from the device path"
    del q_np, out_np
    numpy_line = {"value": round(total_cells / np_s / 1e9, 3), "unit": "Gcells/s",
                  "ms_per_step": round(np_s * 1e3, 2),
                  "path": "paper_2409_07704_b200.align(numpy float32 [B,T,S]) -> numpy uint8, "
                          "pageable host memory (the reference binding's call)"}
    # ---- score export (forward_parallel): Q written in place
    qs = torch.empty_like(q)
    for _ in range(2):
        qs.copy_(q)
        mas.forward_parallel(qs)
    sc_ms = []
    for _ in range(3):
        qs.copy_(q)  # the call overwrites its input; the refill is not timed
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        mas.forward_parallel(qs)
        s1.record()
        torch.cuda.synchronize(dev)
        sc_ms.append(s0.elapsed_time(s1))
    del qs
    sc_best = statistics.median(sc_ms)
    scores_line = {"value": round(total_cells / (sc_best / 1e3) / 1e9, 2), "unit": "Gcells/s",
                   "ms_per_step": round(sc_best, 4), "bytes_per_cell": 8,
                   "path": "forward_parallel(torch CUDA tensor): the parallel engine's score "
                           "table written in place (K1's export variant: Q stored over q by TMA)"}
    # ---- fused log-likelihood + MAS: q from the
    # Glow-TTS prior (C = 80 channels) computed on tcgen05 inside K1, never
    # written; against the unfused pipeline (gaussian_loglik writes q, then
    # the plan aligns it).  Same batch shape as the step, on this rank.
    gauss_line = None
    try:
        C = 80
        gz = torch.Generator(device="cpu").manual_seed(1)
        zz = torch.randn(B, C, S, generator=gz).to(dev)
        mu = (torch.randn(B, C, T, generator=gz) * 0.8).to(dev)
        lsd = ((torch.rand(B, C, T, generator=gz) - 0.5) * 0.6).to(dev)

        def unfused_call():
            qg = mas.gaussian_loglik(zz, mu, lsd)
            plan.enqueue(qg, out, stream=torch.cuda.current_stream(dev))

        gplan = mas.GaussianPlan(B, C, T, S)
        gout = torch.empty_like(out)

        def fused_call():
            gplan.enqueue(zz, mu, lsd, out=gout, stream=torch.cuda.current_stream(dev))

        fused_call()
        unfused_call()
        torch.cuda.synchronize(dev)
        assert torch.equal(gout, out), "fused != unfused alignment"
        checked_out = mas.align_gaussian(zz, mu, lsd)["alignment"]
        assert torch.equal(checked_out, out), "align_gaussian != unfused alignment"
        del checked_out

        def ev_ms(fn, n=5):
            fn()
            torch.cuda.synchronize(dev)
            ts = []
            for _ in range(n):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize(dev)
                ts.append(e0.elapsed_time(e1))
            return statistics.median(ts)

        f_ms, u_ms = ev_ms(fused_call), ev_ms(unfused_call)
        chk_ms = ev_ms(lambda: mas.align_gaussian(zz, mu, lsd), n=3)
        gplan.close()
        del gout
        kp = ((2 * C + 63) // 64) * 64
        gauss_line = {
            "value": round(total_cells / (f_ms / 1e3) / 1e9, 2), "unit": "Gcells/s",
            "ms_per_step": round(f_ms, 4), "unfused_ms_per_step": round(u_ms, 4),
            "speedup_vs_unfused": round(u_ms / f_ms, 3), "channels": C,
            "align_gaussian_checked_ms": round(chk_ms, 4),
            "bytes_per_cell": 1.125,
            "tensor": {"achieved_tflops": round(2 * kp * cells / (f_ms / 1e3) / 1e12, 1),
                       "flops_per_cell": 2 * kp, "peak_tflops": _bf16_peak(),
                       "frac": round(2 * kp * cells / (f_ms / 1e3) / 1e12 / _bf16_peak(), 4)},
            "path": "GaussianPlan.enqueue(z, mean, logstd): operand prep + K1 computing q tiles "
                    "with tcgen05 (bf16 operands, fp32 accumulation) into the DP ring + K2; vs "
                    "gaussian_loglik (q to HBM) + plan.enqueue; both enqueue-only. "
                    "align_gaussian_checked_ms: the one-shot call (plan, workspace, host check)",
        }
        del zz, mu, lsd
    except Exception as e:  # reported, not fatal for the headline line
        gauss_line = {"error": str(e)[:200]}
    durations_line = {
        "value": round(total_cells / (dur_ms / 1e3) / 1e9, 2), "unit": "Gcells/s",
        "ms_per_step": round(dur_ms, 4), "bytes_per_cell": 4.125,
        "frac": None,  # filled below once the peak is known
        "e2e": {"value": round(total_cells * e2e_steps / e2e_dur_s / 1e9, 3),
                "unit": "Gcells/s", "h2d_bytes_per_step": B * T * S * 4,
                "d2h_bytes_per_step": B * T * 4 + 4 * B,
                "path": "mas_align_host_ex (C-ABI), pinned host in, durations out"},
        "path": "plan.enqueue(durations=...): K1 without the zero fill + K2 writing [B,T] int32",
    }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            ms, cores, sample, ref_cells = cpu_reference_leg(20, 1, budget_s=12.0,
                                                             config=args.config)
            cpu = {"value": round(ref_cells * len(ms) / (sum(ms) / 1e3) / 1e9, 4),
                   "unit": "Gcells/s", "cores": cores, "kind": "reference", "sample": sample}
        except Exception as e:  # the reference build did not travel
            cpu = {"value": None, "unit": "Gcells/s", "cores": None, "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    peak, peak_src = _peaks()
    fwd_avg = statistics.mean(fwd_ms)
    bt_avg = statistics.mean(bt_ms)
    achieved = BYTES_PER_CELL * cells / (fwd_avg / 1e3) / 1e9
    traffic = _ncu_traffic()
    step_ms = elapsed_ms / K
    durations_line["frac"] = round(4.125 * cells / (durations_line["ms_per_step"] / 1e3) / 1e9
                                   / peak, 4)
    scores_line["frac"] = round(8 * cells / (scores_line["ms_per_step"] / 1e3) / 1e9 / peak, 4)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "Gcells/s", "n_gpus": world,
        "steps": K, "warmup": max(args.warmup, 3), "ms_per_step": round(step_ms, 4),
        "higher_is_better": True, "scaling": c["scaling"], "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (bench::generate_random_batch seed 0, generated bit-identically on "
                "the device)",
        "config": workload_config(args.config, world),
        "parallelism": f"batch-shard dp{world}, no collective; rank 0 items [{b0}, {b1})",
        "pipelining": "steady state of back-to-back batches: batch k's backtrack (K2) overlaps "
                      "batch k+1's forward (K1) via programmatic dependent launch "
                      "(Plan(pipelined=True)); every batch runs K1+K2 in full",
        "latency_ms": round(latency_ms, 4),
        "geometry": geom,
        "roofline": {"bound": "hbm", "kernel": "mas_fwd4_kernel", "achieved": round(achieved, 1),
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "bytes_per_cell": BYTES_PER_CELL,
                     "fwd_ms": round(fwd_avg, 4), "backtrack_ms": round(bt_avg, 4),
                     "step_frac": round(BYTES_PER_CELL * cells / (step_ms / 1e3) / 1e9 / peak, 4)},
        "e2e": {"value": round(e2e_value, 3), "unit": "Gcells/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "roofline": {"bound": "pcie_h2d", "achieved_h2d_GBs":
                             round(h2d * e2e_value / (total_cells / 1e9) / 1e9, 2),
                             "peak_h2d_GBs": round(h2d_gbs, 2),
                             "frac": round(h2d * e2e_value / (total_cells / 1e9) / 1e9 / h2d_gbs, 4),
                             "peak_source": "pinned torch copy of the same bytes, measured here"},
                "path": "mas_align_host (C-ABI), pinned host in/out, H2D+kernels+D2H+checks"},
        "gpu_launches": K * launches_per_step,
        "variants": {"durations_only": durations_line, "numpy_e2e": numpy_line,
                     "score_export": scores_line, "gaussian_fused": gauss_line},
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    return 0


def relaunch_under_torchrun(argv, nproc):
    """`--gpus N` without torchrun's environment: run this script again as N
    ranks (one per GPU) through torch.distributed.run on 127.0.0.1."""
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + list(argv)
    return subprocess.run(cmd).returncode


def spawn_selftest(args):
    """CPU check of the launch path (tests/test_bench_launch.py): every rank
    joins a gloo group, the max-over-ranks reduction runs, rank 0 prints the
    world it saw."""
    import torch
    import torch.distributed as dist

    rank, world, _ = _dist()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.destroy_process_group()
    b0, b1 = rank_items(args.config, rank, world)
    if rank == 0:
        print(json.dumps({"n_gpus": world, "max_over_ranks": float(t.item()),
                          "rank0_items": [b0, b1],
                          "config": workload_config(args.config, world)}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--spawn-selftest", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(sys.argv[1:], args.gpus)
    if args.spawn_selftest:
        return spawn_selftest(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
