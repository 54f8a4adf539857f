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
               "h2d_bytes_per_step": int(raw_h.numel() * 2), "d2h_bytes_per_step": int(img_h.numel()),
               "frames_per_step": E, "api": "paper_1711_06127_b200.pipeline.HostPipeline"}

    cpu_baseline = None
    secondary = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r, cores, sample = oracle_frame_rate(w, raw[0].cpu().numpy(), 12.0)
        cpu_baseline = {"value": r, "unit": "frames/s", "cores": cores, "kind": "oracle", "sample": sample}
    if not args.no_secondary:
        secondary = secondary_3d(local, world, rank)
        secondary.update(secondary_paper3d(local, world, rank))
        secondary.update(secondary_sector(local, world, rank))
        secondary.update(secondary_table1(local, world, rank))

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
            "clocks": clocks, "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    bf.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def secondary_3d(dev_index: int, world: int = 1, rank: int = 0, vols: int = 8):
    """Volumes/s on C4b (3D 32x32 matrix probe, 64x64 lines, 4x4 multi-line,
    pyramid scan conversion to 256^3, u8 line image and volume):
      * "C4b_stream": ``vols`` volumes per call on every rank (C5's batched 3D
        stream; one 1 GiB volume synthesised and replicated -- DAS cost is
        data-independent), value = all ranks' volumes / max-over-ranks time;
      * "C4b_single": ONE volume per call, latency mode: the
        scanlines are split into event-aligned blocks over the ranks
        (dist.ShardedVolume: DAS+envelope per block, all-reduce(max) of the
        frame max, log compression, NCCL all-gather of the u8 line volume),
        rank 0 scan-converts.  At N=1 it is the plain single-GPU call.
    Device-timed with CUDA events, inputs resident in HBM (> L2)."""
    import torch
    import torch.distributed as dist
    import synth
    from synth import configs
    from paper_1711_06127_b200 import SupraBF
    from paper_1711_06127_b200.dist import ShardedVolume
    out = {}
    w = configs.CONFIGS["C4b"]().replace(sc_output_type=configs.T_U8, line_output_type=configs.T_U8)
    dev = torch.device(f"cuda:{dev_index}")
    raw = torch.empty((vols, w.num_events, w.C, w.S), dtype=torch.int16, device=dev)
    synth.channel_data_gpu(w, raw[0], realisation=0)
    for v in range(1, vols):
        raw[v].copy_(raw[0])
    bf = SupraBF(w, device=dev_index, max_frames=vols)
    li, img = bf.empty_line_img(vols), bf.empty_img(vols)

    def timed(fn, reps):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / reps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    def stream_call():
        bf.beamform(raw, vols, line_img=li)
        bf.scanconvert(li, vols, img)

    ms = timed(stream_call, 5)
    out["C4b_stream"] = {"value": vols * world * 1000.0 / ms, "unit": "volumes/s", "ms_per_call": ms,
                         "volumes_per_call_per_rank": vols, "scaling": "weak"}

    sv = ShardedVolume(bf, w.L, w.S, torch.uint8, dev, align=4 * w.num_lines_x)

    def single_call():
        y = sv.run(raw[:1])
        if rank == 0:
            bf.scanconvert(y, 1, img)

    ms = timed(single_call, 10)
    out["C4b_single"] = {"value": 1000.0 / ms, "unit": "volumes/s", "ms_per_volume": ms,
                         "volumes_per_call": 1, "scaling": "strong",
                         "parallelism": f"scanline blocks x{world}, all-reduce(max) + all-gather u8 line volume"
                         if world > 1 else "single GPU"}
    bf.close()
    del raw, li, img, sv
    torch.cuda.empty_cache()
    return out


def secondary_paper3d(dev_index: int, world: int = 1, rank: int = 0, vols: int = 4):
    """Volumes/s on the paper's own 3D shape (C4p: 32x32 matrix probe through
    384 channels, 32x16 scanlines, 60 deg, 70 mm, 0.175 mm pyramid output
    401x401x402 u8): "C4p_single" one volume per
    call, "C4p_stream" ``vols`` volumes per call per rank (weak scaling).
    DAS + envelope/log + scan conversion, device-timed, inputs resident."""
    import torch
    import torch.distributed as dist
    import synth
    from synth import configs
    from paper_1711_06127_b200 import SupraBF
    dev = torch.device(f"cuda:{dev_index}")
    w = configs.c4p(sc_output_type=configs.T_U8, line_output_type=configs.T_U8)
    raw = torch.empty((vols, w.num_events, w.C, w.S), dtype=torch.int16, device=dev)
    synth.channel_data_gpu(w, raw[0], realisation=0)
    for v in range(1, vols):
        raw[v].copy_(raw[0])
    bf = SupraBF(w, device=dev_index, max_frames=vols)
    li, img = bf.empty_line_img(vols), bf.empty_img(vols)
    out = {}
    for n, key, reps in ((1, "C4p_single", 10), (vols, "C4p_stream", 5)):
        def call():
            bf.beamform(raw, n, line_img=li)
            bf.scanconvert(li, n, img)
        for _ in range(2):
            call()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            call()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / reps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
        out[key] = {"value": n * world * 1000.0 / ms, "unit": "volumes/s", "ms_per_call": ms,
                    "volumes_per_call_per_rank": n, "scaling": "weak",
                    "paper_gtx1080_vol_s_context": round(1000 / 27.49, 1)}
    bf.close()
    del raw, li, img
    torch.cuda.empty_cache()
    return out


def secondary_sector(dev_index: int, world: int = 1, rank: int = 0, frames: int = 16):
    """Frames/s on BASELINE.json configs[2] = C3: phased 128-element probe,
    192 steered lines over 60 deg, 4096 samples, sector scan conversion to
    512 x 512 u8; ``frames`` per call per rank (the config's 16-frame
    batch), DAS + envelope/log + scan conversion, device-timed."""
    import torch
    import torch.distributed as dist
    from synth import configs
    from paper_1711_06127_b200 import SupraBF
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from gpu_util import raw_frames
    dev = torch.device(f"cuda:{dev_index}")
    w = configs.c3(sc_output_type=configs.T_U8)
    raw = raw_frames(w, frames, device=dev)
    bf = SupraBF(w, device=dev_index, max_frames=frames)
    li, img = bf.empty_line_img(frames), bf.empty_img(frames)

    def call():
        bf.beamform(raw, frames, line_img=li)
        bf.scanconvert(li, frames, img)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        call()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / 10], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    bf.close()
    del raw, li, img
    torch.cuda.empty_cache()
    return {"C3": {"value": frames * world * 1000.0 / ms, "unit": "frames/s", "ms_per_call": ms,
                   "frames_per_call_per_rank": frames, "scaling": "weak"}}


# The paper's own 2D benchmark rows (Table 1): GeForce GTX 1080
# total node run-time per frame -> frames/s, quoted as context only.
PAPER_T1_GTX1080_FPS = {"T1_64_1": 1000 / 5.37, "T1_64_2": 1000 / 4.24, "T1_128_1": 1000 / 4.38,
                        "T1_128_2": 1000 / 5.00}


def secondary_table1(dev_index: int, world: int = 1, rank: int = 0, frames: int = 64):
    """Frames/s on the paper's Table-1 2D shapes:
    128-element linear probe with 64 receive channels (walking aperture),
    (transmit events / multi-line) = 64/1, 64/2, 128/1, 128/2, 45 mm depth,
    u8 B-mode on the 0.0225 mm grid.  ``frames`` per call on every rank
    (weak scaling), DAS + envelope/log + scan conversion, device-timed with
    CUDA events, inputs resident in HBM."""
    import torch
    import torch.distributed as dist
    from synth import configs
    from paper_1711_06127_b200 import SupraBF
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from gpu_util import raw_frames
    dev = torch.device(f"cuda:{dev_index}")
    out = {}
    for name, paper_fps in PAPER_T1_GTX1080_FPS.items():
        w = configs.CONFIGS[name](sc_output_type=configs.T_U8, line_output_type=configs.T_U8)
        raw = raw_frames(w, frames, device=dev)
        bf = SupraBF(w, device=dev_index, max_frames=frames)
        li, img = bf.empty_line_img(frames), bf.empty_img(frames)

        def call():
            bf.beamform(raw, frames, line_img=li)
            bf.scanconvert(li, frames, img)
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        a.record()
        for _ in range(reps):
            call()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / reps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
        out[name] = {"value": frames * world * 1000.0 / ms, "unit": "frames/s", "ms_per_call": ms,
                     "frames_per_call_per_rank": frames, "lines": w.L, "channels": w.C,
                     "scaling": "weak", "paper_gtx1080_fps_context": round(paper_fps, 1)}
        bf.close()
        del raw, li, img
        torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    sys.exit(main())
