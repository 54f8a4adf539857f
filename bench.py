#!/usr/bin/env python
"""Benchmark: beamformed frames/s of the DAS -> envelope/log -> scan-conversion
hot path (BASELINE.json metric) on configs[1] = C2 (2D linear array, 128
channels, 256 scanlines, 2048 samples, 100-frame speckle stream).

One step = one pass of the whole hot path over one batch of 100 frames
(inputs resident in HBM): supra_bf_beamform (DAS + fused envelope/log +
frame-max finalisation) and supra_bf_scanconvert (u8 B-mode, 1694 x 1752),
plus, for N > 1 GPUs, the NCCL gather of every rank's B-mode images to rank 0.

  python bench.py [--gpus N --steps K --warmup W]          # our CUDA path
  python bench.py --impl reference [...]                    # the CPU oracle

Prints one JSON line (rank 0).  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "beamformed frames/s (2D) and volumes/s (3D) at 1/2/4/8 B200; DAS HBM GB/s vs peak"
WORKLOAD_DESC = {
    "C2": "C2: 2D linear array, 128 channels, 256 scanlines, 2048 samples/channel, int16, "
          "100-frame stream (4 speckle realisations cycled), u8 B-mode 1694x1752",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=int, default=None, help="frames per step (default: the config's)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.tmp,
                stderr=subprocess.DEVNULL)
        except (OSError, ValueError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.tmp.flush()
        self.tmp.seek(0)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.tmp.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.tmp.name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_traffic(config: str, frames: int):
    """DRAM bytes per DAS launch from the committed ncu capture (profiles/)."""
    try:
        with open(os.path.join(ROOT, "profiles", "das_ncu.json")) as f:
            d = json.load(f)
        e = d.get(config, {})
        if e.get("frames") == frames:
            return e["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        pass
    return None


# ------------------------------------------------------------------ oracle (reference arm / cpu baseline)
def oracle_frame_rate(w, raw_np, seconds_budget: float):
    """Time the oracle (as it stands) on a bounded sample of the workload:
    DAS + IQ envelope + log compression of a block of scanlines of one
    frame, plus scan conversion of the same fraction of output rows
    (all host cores; the oracle threads DAS over lines).  Returns
    (frames/s, cores, sample description)."""
    import numpy as np
    import oracle
    cores = os.cpu_count() or 1
    L = w.L
    # calibrate with a small block
    t0 = time.perf_counter()
    nl = max(1, min(L, cores))
    lines = np.arange(nl, dtype=np.int32)
    rf = oracle.das(w, raw_np, lines=lines, nthreads=cores)
    env = oracle.envelope(w, rf)
    oracle.log_compress(env, w.dynamic_range_db)
    per_line = (time.perf_counter() - t0) / nl
    nl = int(max(1, min(L, seconds_budget * 0.8 / max(per_line, 1e-6))))
    nl = max(cores, (nl // cores) * cores) if nl >= cores else nl
    nl = min(nl, L)
    # whole frames fit the budget: repeat the full frame (bounded, <= 100)
    nrep = 1
    if nl == L:
        nrep = int(max(1, min(100, seconds_budget * 0.8 / max(per_line * L, 1e-6))))
    lines = np.arange(nl, dtype=np.int32)
    # scan conversion sample: the same fraction of the output rows
    frac = nl / L
    sw = w.replace(out_dims=(w.out_dims[0], w.out_dims[1], max(1, int(round(w.out_dims[2] * frac)))))
    t0 = time.perf_counter()
    for _ in range(nrep):
        rf = oracle.das(w, raw_np, lines=lines, nthreads=cores)
        env = oracle.envelope(w, rf)
        y, _ = oracle.log_compress(env, w.dynamic_range_db)
        yfull = np.zeros((L, w.S))
        yfull[:nl] = y
        oracle.scan_convert(sw, yfull)
    dt = time.perf_counter() - t0
    rate = nrep * frac / dt
    sample = (f"{nrep} x {nl}/{L} scanlines of one {w.name} frame (DAS {cores} threads + IQ envelope + log) "
              f"+ scan conversion of {sw.out_dims[2]}/{w.out_dims[2]} output rows; {dt:.2f} s")
    return rate, cores, sample


def run_reference(args):
    """--impl reference: the CPU oracle timed on the box's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    import synth
    from synth import configs
    w = configs.CONFIGS[args.config]()
    raw_np = synth.channel_data_cpu(w.replace(num_events=w.num_events), realisation=0) \
        if w.raw_bytes_per_frame() < (64 << 20) else _gpu_or_cpu_frame(w)
    total_budget = 90.0
    per_step = total_budget / max(1, args.steps + args.warmup)
    rates = []
    sample = ""
    cores = os.cpu_count() or 1
    for i in range(args.warmup + args.steps):
        r, cores, sample = oracle_frame_rate(w, raw_np, per_step)
        if i >= args.warmup:
            rates.append(r)
    value = statistics.median(rates) if rates else 0.0
    line = {"metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value if value else None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": WORKLOAD_DESC.get(args.config, args.config), "frames_per_step": "sample"},
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _gpu_or_cpu_frame(w):
    """One frame of the workload on the host (GPU synthesis when available)."""
    import synth
    try:
        import torch
        if torch.cuda.is_available():
            t = torch.empty((w.num_events, w.C, w.S), dtype=torch.int16, device="cuda")
            synth.channel_data_gpu(w, t, realisation=0)
            return t.cpu().numpy()
    except Exception:
        pass
    return synth.channel_data_cpu(w)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from synth import configs
    from paper_1711_06127_b200 import SupraBF
    from paper_1711_06127_b200.dist import OverlappedGather
    from paper_1711_06127_b200.pipeline import HostPipeline

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")

    w = configs.CONFIGS[args.config]().replace(sc_output_type=configs.T_U8)
    F = args.frames or w.frames
    nreal = min(F, w.realisations)
    raw = torch.empty((F, w.num_events, w.C, w.S), dtype=torch.int16, device=dev)
    for r in range(nreal):
        synth.channel_data_gpu(w, raw[r], realisation=r)
    for f in range(nreal, F):
        raw[f].copy_(raw[f % nreal])
    torch.cuda.synchronize()

    bf = SupraBF(w, device=local, max_frames=F)
    info = bf.info()
    li = bf.empty_line_img(F)
    img = bf.empty_img(F)
    nx, ny, nz = w.out_dims
    # N > 1: the u8 B-mode batch of step i is gathered to rank 0 (NCCL) while
    # step i + 1 beamforms (double-buffered images, stream-ordered waits)
    gat = OverlappedGather(img, dst=0)
    stream = torch.cuda.current_stream(dev)
    nstep = [0]

    def step():
        i = nstep[0]
        nstep[0] += 1
        out = gat.buffer(i)
        bf.beamform(raw, F, line_img=li)
        bf.scanconvert(li, F, out)
        gat.submit(i)

    for _ in range(max(3, args.warmup)):
        step()
    gat.drain()
    torch.cuda.synchronize()

    K = args.steps
    das_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b in das_ev:      # created + marked recorded; the library re-records them around DAS
        a.record(stream)
        b.record(stream)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    try:
        clk_id = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)
    except Exception:
        clk_id = str(local)
    clk = ClockSampler(clk_id)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.start()
    time.sleep(0.2)
    start.record(stream)
    for i in range(K):
        bf.set_das_events(*das_ev[i])
        step()
    gat.drain()          # the last gathers belong to the timed steps
    stop.record(stream)
    torch.cuda.synchronize()
    bf.set_das_events(None, None)
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = start.elapsed_time(stop)
    das_ms = sum(a.elapsed_time(b) for a, b in das_ev) / K
    t = torch.tensor([ms, das_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, das_ms = float(t[0]), float(t[1])
    ms_per_step = ms / K
    value = F * world * K / (ms / 1000.0)

    # roofline of the dominant kernel (das_fused): algorithmic bytes per launch
    alg_bytes = (info["referenced_bytes_per_frame"] + w.L * w.S * 4) * F
    peak, peak_kind = measured_peak_hbm()
    achieved = alg_bytes / (das_ms / 1000.0) / 1e9
    traffic = ncu_traffic(args.config, F)
    roofline = {"bound": "hbm", "kernel": "das_fused", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                "das_ms_per_launch": das_ms, "algorithmic_bytes_per_launch": alg_bytes,
                "das_share_of_step": das_ms / ms_per_step}
    roofline.update(counter_extras(info, F, das_ms, args.config, achieved))

    # N > 1: the same stream without the gather (per-rank
    # compute rate) and with the line-domain variant (u8 line images, 0.5 MB
    # per C2 frame instead of the 2.97 MB B-mode, gathered to rank 0; scan
    # conversion then happens where the images are displayed)
    multi = None
    if world > 1:
        def timed_steps(fn, k):
            for j in range(3):
                fn(j)
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for j in range(k):
                fn(3 + j)
            b.record(stream)
            torch.cuda.synchronize()
            dist.barrier()
            tt = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return float(tt[0])

        def step_ng(_):
            bf.beamform(raw, F, line_img=li)
            bf.scanconvert(li, F, img)
        ms_ng = timed_steps(step_ng, K)
        bf8 = SupraBF(w.replace(line_output_type=configs.T_U8), device=local, max_frames=F)
        g8 = OverlappedGather(bf8.empty_line_img(F), dst=0)

        def step_ld(j):
            bf8.beamform(raw, F, line_img=g8.buffer(j))
            g8.submit(j)

        def step_ld_drained(j):
            step_ld(j)
            if j == 3 + K - 1:
                g8.drain()
        ms_ld = timed_steps(step_ld_drained, K)
        bf8.close()
        multi = {"no_gather": {"value": F * world * K / (ms_ng / 1000.0), "unit": "frames/s",
                               "ms_per_step": ms_ng / K,
                               "what": "beamform + scanconvert on every rank, no collective"},
                 "line_domain_gather": {"value": F * world * K / (ms_ld / 1000.0), "unit": "frames/s",
                                        "ms_per_step": ms_ld / K,
                                        "what": "beamform to u8 line images + NCCL gather of the line "
                                                "images to rank 0 (no scan conversion)"}}

    # end to end: pinned host input -> public API (HostPipeline) -> pinned host B-mode
    e2e = None
    if not args.no_e2e:
        E = min(F, 16)
        raw_h = raw[:E].cpu().pin_memory()
        img_h = torch.empty((E, nz, ny, nx), dtype=torch.uint8).pin_memory()
        pipe = HostPipeline(bf, chunk=4, device=local)
        pipe.run(raw_h, img_h)
        reps = 3
        t0 = time.perf_counter()
        for _ in range(reps):
            pipe.run(raw_h, img_h)
        dt = (time.perf_counter() - t0) / reps
        rate = torch.tensor([E / dt], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(rate, op=dist.ReduceOp.MIN)
        e2e = {"value": float(rate) * world, "unit": "frames/s",
               "h2d_bytes_per_step": int(pipe.h2d_bytes), "d2h_bytes_per_step": int(img_h.numel()),
               "frames_per_step": E, "api": "paper_1711_06127_b200.pipeline.HostPipeline",
               "h2d": "supra_bf_stage_raw: the device reads the referenced sample ranges of each "
                      "pinned host frame over PCIe (%.0f %% of the %d-byte frame)"
                      % (100.0 * pipe.h2d_bytes / max(1, raw_h.numel() * 2), raw_h[0].numel() * 2)}

    cpu_baseline = None
    secondary = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r, cores, sample = oracle_frame_rate(w, raw[0].cpu().numpy(), 12.0)
        cpu_baseline = {"value": r, "unit": "frames/s", "cores": cores, "kind": "oracle", "sample": sample}
    if not args.no_secondary:
        secondary = secondary_all(local, world, rank)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": K,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 (int16 input)", "data": "synthetic",
            "config": {"workload": WORKLOAD_DESC.get(args.config, args.config), "frames_per_step": F,
                       "frames_per_cta": info["frames_per_cta"],
                       "l2": "inputs 12.8 GiB per step > 126 MB L2 (no flush needed)",
                       "parallelism": f"frames x{world} (weak), NCCL gather of u8 B-mode to rank 0"
                       if world > 1 else "single GPU"},
            "roofline": roofline, "cpu_baseline": cpu_baseline, "e2e": e2e,
            "gpu_launches": K * (info["kernels_per_beamform"] + info["kernels_per_scanconvert"]),
            "clocks": clocks, "multi_gpu": multi, "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    bf.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


# B200 unit counts for the ALU roofline (B200_PROFILING.md / the CUDA
# throughput tables): 4 warp schedulers per SM each issue one warp
# instruction per clock, 148 SMs, at the max SM clock.
ISSUE_PEAK_WARP_INST_S = 148 * 4 * 1.965e9


def ncu_entry(key: str, frames: int):
    """The committed ncu capture (profiles/das_ncu.json) of config ``key``'s
    DAS launch at ``frames`` frames per call, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "das_ncu.json")) as f:
            e = json.load(f).get(key, {})
        return e if e.get("frames") == frames else None
    except (OSError, ValueError):
        return None


def counter_extras(info: dict, frames: int, das_ms: float, key: str, achieved_gbs=None):
    """SURVEY 8(d)'s per-kernel report beside the roofline: Gtaps/s, the
    fraction of the issue ceiling (warp instructions of the same launch shape
    from profiles/das_ncu.json over the live DAS time), the fraction of the
    nominal 8 TB/s, and the L1 / L2 sector hit rates of the ncu capture."""
    out = {"gtaps_per_s": info["taps_per_frame"] * frames / (das_ms / 1000.0) / 1e9}
    if achieved_gbs is not None:
        out["frac_of_nominal_8tbs"] = achieved_gbs / 8000.0
    e = ncu_entry(key, frames)
    if e:
        if e.get("warp_inst_per_launch"):
            out["issue_frac"] = e["warp_inst_per_launch"] / (das_ms / 1000.0) / ISSUE_PEAK_WARP_INST_S
        for k in ("l2_hit_rate", "l1_hit_rate"):
            if k in e:
                out[k] = e[k]
    return out


def hbm_roofline(info: dict, frames: int, L: int, Sd: int, das_ms: float, key: str):
    """DAS HBM roofline: algorithmic bytes = referenced int16 input (distinct
    samples any tap reads, host-counted at create) + the f32 envelope written
    (frame-max mode), per call, over the DAS launches' CUDA-event time."""
    alg = (info["referenced_bytes_per_frame"] + L * Sd * 4) * frames
    peak, kind = measured_peak_hbm()
    ach = alg / (das_ms / 1000.0) / 1e9
    e = ncu_entry(key, frames)
    out = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
           "traffic": e.get("dram_bytes_per_launch") if e else None, "peak_kind": peak_kind_str(kind),
           "das_ms_per_call": das_ms, "algorithmic_bytes_per_call": alg}
    out.update(counter_extras(info, frames, das_ms, key, ach))
    return out


def alu_roofline(info: dict, frames: int, das_ms: float, key: str):
    """DAS ALU (issue) roofline for the multi-line shapes (M > 1: each input
    sample feeds several lines, SURVEY 8(d) "ALU-bound"): warp instructions
    the DAS launches issue per call (ncu smsp__inst_executed.sum of the same
    launch shape, profiles/das_ncu.json) over their CUDA-event time, against
    the issue peak 148 SMs x 4 schedulers x 1.965 GHz.  Also reported: taps/s
    (taps = (line, sample, aperture member) triples per frame x frames)."""
    taps = info["taps_per_frame"] * frames
    out = {"bound": "alu", "unit": "warp-inst/s", "peak": ISSUE_PEAK_WARP_INST_S,
           "peak_kind": "derived: 148 SMs x 4 issue/clk x 1.965 GHz (B200_PROFILING.md unit counts)",
           "taps_per_s": taps / (das_ms / 1000.0), "das_ms_per_call": das_ms,
           "hbm_frac": (info["referenced_bytes_per_frame"] * frames / (das_ms / 1000.0) / 1e9)
           / measured_peak_hbm()[0]}
    e = ncu_entry(key, frames)
    if e and e.get("warp_inst_per_launch"):
        ach = e["warp_inst_per_launch"] / (das_ms / 1000.0)
        out.update({"achieved": ach, "frac": ach / ISSUE_PEAK_WARP_INST_S,
                    "warp_inst_per_call": e["warp_inst_per_launch"],
                    "inst_source": "profiles/das_ncu.json (ncu --set full)"})
    else:
        out.update({"achieved": None, "frac": None})
    out.update({k: v for k, v in counter_extras(info, frames, das_ms, key).items() if k in ("l2_hit_rate", "l1_hit_rate")})
    return out


def peak_kind_str(kind: str) -> str:
    return "measured (MEASURED_PEAKS.json hbm_gbs)" if kind == "measured" else kind


def _timed_calls(bf, fn, reps: int, world: int, dev):
    """(ms per call, DAS ms per call): CUDA events around the calls on the
    current stream and the library's DAS events around each call's DAS
    launches, after 2 warm-up calls; max over ranks."""
    import torch
    import torch.distributed as dist
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    st = torch.cuda.current_stream(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for x, y in evs:
        x.record(st)
        y.record(st)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for i in range(reps):
        bf.set_das_events(*evs[i])
        fn()
    b.record(st)
    torch.cuda.synchronize()
    bf.set_das_events(None, None)
    t = torch.tensor([a.elapsed_time(b) / reps, sum(x.elapsed_time(y) for x, y in evs) / reps],
                     dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0]), float(t[1])


def _volumes(w, n, dev, distinct=4):
    """n frames/volumes on the device: realisations 0..distinct-1 (distinct
    noise / speckle), cycled.  DAS cost does not depend on the data."""
    import torch
    import synth
    out = torch.empty((n, w.num_events, w.C, w.S), dtype=torch.int16, device=dev)
    k = max(1, min(n, distinct))
    for v in range(k):
        synth.channel_data_gpu(w, out[v], realisation=v)
    for v in range(k, n):
        out[v].copy_(out[v % k])
    return out


def secondary_line(key: str, w, n: int, reps: int, dev_index: int, world: int, unit: str, bound: str,
                   extra=None):
    """One device-timed secondary line: ``n`` frames/volumes per call on every
    rank (weak scaling), DAS + envelope/log + scan conversion (u8 line image
    and B-mode, frame-max reference), inputs resident in HBM; value = all
    ranks' units / max-over-ranks time; roofline of the DAS launches."""
    import torch
    from paper_1711_06127_b200 import SupraBF
    dev = torch.device(f"cuda:{dev_index}")
    raw = _volumes(w, n, dev)
    bf = SupraBF(w, device=dev_index, max_frames=n)
    li, img = bf.empty_line_img(n), bf.empty_img(n)
    info = bf.info()

    def call():
        bf.beamform(raw, n, line_img=li)
        bf.scanconvert(li, n, img)
    ms, das_ms = _timed_calls(bf, call, reps, world, dev)
    Sd = w.S // max(1, w.decimation)
    roof = (hbm_roofline(info, n, w.L, Sd, das_ms, key) if bound == "hbm"
            else alu_roofline(info, n, das_ms, key))
    out = {"value": n * world * 1000.0 / ms, "unit": unit, "ms_per_call": ms,
           "per_call_per_rank": n, "scaling": "weak", "das_ms_per_call": das_ms,
           "das_share": das_ms / ms, "frames_per_cta": info["frames_per_cta"], "roofline": roof,
           "input_gib_per_call": round(n * w.raw_bytes_per_frame() / 2 ** 30, 3)}
    if extra:
        out.update(extra)
    bf.close()
    del raw, li, img
    torch.cuda.empty_cache()
    return out


def secondary_all(dev_index: int, world: int, rank: int):
    from synth import configs
    u8 = dict(sc_output_type=configs.T_U8, line_output_type=configs.T_U8)
    ctx3d = {"paper_gtx1080_vol_s_context": round(1000 / 27.49, 1)}
    out = {}
    # 3D, 32x32 matrix probe, 64x64 lines, 2048 samples, pyramid 256^3
    out["C4a_single"] = secondary_line("C4a", configs.c4("a", **u8), 1, 5, dev_index, world, "volumes/s",
                                       "hbm", {"lines": 4096, "events": 4096,
                                               "note": "M = 1: 16 GiB of int16 per volume, HBM-bound"})
    # the same volumes streamed two per call (32 GiB of input per call): the
    # mirror-quad CTAs take both volumes, sharing each tap's geometry by 8
    out["C4a_stream"] = secondary_line("C4a_stream", configs.c4("a", **u8), 2, 5, dev_index, world, "volumes/s",
                                       "hbm", {"lines": 4096, "events": 4096,
                                               "note": "M = 1, 2 volumes per call: HBM-bound"})
    out["C4b_stream"] = secondary_line("C4b", configs.c4("b", **u8), 8, 5, dev_index, world, "volumes/s",
                                       "alu", {"note": "4x4 multi-line (each sample feeds 16 lines): ALU-bound"})
    out["C4b_single"] = secondary_c4b_single(dev_index, world, rank)
    # the paper's 3D row: 384 channels, 32x16 lines, 70 mm, 401x401x402
    out["C4p_single"] = secondary_line("C4p_1", configs.c4p(**u8), 1, 10, dev_index, world, "volumes/s",
                                       "hbm", ctx3d)
    out["C4p_stream"] = secondary_line("C4p", configs.c4p(**u8), 4, 5, dev_index, world, "volumes/s",
                                       "hbm", ctx3d)
    # BASELINE configs[2]: phased 128 el, 192 lines, 4096 samples, sector 512^2;
    # 32 frames per call (SURVEY 8(d) protocol: 2D >= 25 frames per call)
    out["C3"] = secondary_line("C3", configs.c3(sc_output_type=configs.T_U8), 32, 10, dev_index, world,
                               "frames/s", "hbm")
    for name, fps in PAPER_T1_GTX1080_FPS.items():
        out[name] = secondary_line(name, configs.CONFIGS[name](**u8), 64, 10, dev_index, world, "frames/s",
                                   "hbm" if name.endswith("_1") else "alu",
                                   {"paper_gtx1080_fps_context": round(fps, 1)})
    return out


def secondary_c4b_single(dev_index: int, world: int, rank: int):
    """ONE C4b volume per call, latency mode: the scanlines
    are split into event-aligned blocks over the ranks (dist.ShardedVolume:
    DAS+envelope per block, all-reduce(max) of the frame max, log
    compression, NCCL all-gather of the u8 line volume), rank 0
    scan-converts.  At N=1 it is the single-GPU call."""
    import torch
    from synth import configs
    from paper_1711_06127_b200 import SupraBF
    from paper_1711_06127_b200.dist import ShardedVolume
    w = configs.c4("b", sc_output_type=configs.T_U8, line_output_type=configs.T_U8)
    dev = torch.device(f"cuda:{dev_index}")
    raw = _volumes(w, 1, dev)
    bf = SupraBF(w, device=dev_index, max_frames=1)
    img = bf.empty_img(1)
    info = bf.info()
    sv = ShardedVolume(bf, w.L, w.S, torch.uint8, dev, align=4 * w.num_lines_x)

    def call():
        y = sv.run(raw)
        if rank == 0:
            bf.scanconvert(y, 1, img)
    ms, das_ms = _timed_calls(bf, call, 10, world, dev)
    out = {"value": 1000.0 / ms, "unit": "volumes/s", "ms_per_volume": ms, "volumes_per_call": 1,
           "scaling": "strong", "das_ms_per_call": das_ms, "roofline": alu_roofline(info, 1, das_ms, "C4b_1"),
           "parallelism": f"scanline blocks x{world}, all-reduce(max) + all-gather u8 line volume"
           if world > 1 else "single GPU"}
    bf.close()
    del raw, img, sv
    torch.cuda.empty_cache()
    return out


# The paper's own 2D benchmark rows (Table 1): GeForce GTX 1080
# total node run-time per frame -> frames/s, quoted as context only.
PAPER_T1_GTX1080_FPS = {"T1_64_1": 1000 / 5.37, "T1_64_2": 1000 / 4.24, "T1_128_1": 1000 / 4.38,
                        "T1_128_2": 1000 / 5.00}


if __name__ == "__main__":
    sys.exit(main())
