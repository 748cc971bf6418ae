"""Stage-I stabilization throughput on B200 (BASELINE.json metric:
"stabilized frames/s at 1080p (1/2/4/8 B200); kernel % of HBM roofline").

One step = stabilizing the whole configs[2] sequence (1920x1080 RGB as
BT.601 Y/Cb/Cr 4:4:4, 1000 frames, similarity, 1000 corners, RANSAC 500 @ 3
px, smoothing radius 30).  `value` is device-resident throughput (inputs in
HBM before the timed region; 6.2 GB of input per step, far larger than L2);
`e2e` is the same step through the C-ABI host-buffer entry point
(stabgpu_stabilize_sequence) with pinned-host input and output copied inside
the timed region.  N > 1 (torchrun): contiguous re-detect-aligned frame
shards per rank, one all-gather of ~100 B/frame motion records, every rank
composes its own frames.

--impl reference times the reference's own CPU implementation (the
unmodified reference sources compiled into oracle/_ref, driven segment-
parallel on all host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "stabilized frames/s at 1080p (1/2/4/8 B200); kernel % of HBM roofline"
UNIT = "frames/s"


def compose_traffic(spec, planes, frames):
    """DRAM bytes (read + write) of one compose launch, from the committed ncu
    --set full capture (profiles/compose_traffic.json), scaled per frame."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "compose_traffic.json")
    try:
        t = json.load(open(p))
    except (OSError, ValueError):
        return None
    if (t["width"], t["height"], t["planes"]) != (spec.width, spec.height, planes):
        return None
    return (t["dram_bytes_read"] + t["dram_bytes_write"]) * frames / t["frames_per_launch"]


def kernel_rooflines(spec, stab_cfg, frames, c, hbm):
    """HBM fraction of the other bandwidth-class stages (north_star: pyramid,
    corner and warp kernels).  Algorithmic bytes per SURVEY.md 8(d):
    K1 = W*H + sum_{l>=1} W_l*H_l per frame (read the base once, write each
    level once); K2/K3 = 2 (W_roi+4)(H_roi+4) per detection frame (response
    pass + exact pass; the stage time also holds K4's greedy select)."""
    if frames <= 0:
        return None
    from paper_1701_03572_b200 import stab

    w, h = spec.width, spec.height
    pyr = w * h
    lw, lh = w, h
    for _ in range(1, stab_cfg.flow.max_levels):
        if lw // 2 < 16 or lh // 2 < 16:  # image_ops.cpp:71
            break
        lw, lh = lw // 2, lh // 2
        pyr += lw * lh
    roi = stab.detection_roi((h, w), stab_cfg.detect.roi_margin)
    ndet = (frames - 1 + stab_cfg.flow.redetect_interval - 1) // stab_cfg.flow.redetect_interval
    det = 2 * (roi.x1 - roi.x0 + 4) * (roi.y1 - roi.y0 + 4)
    out = {}
    for name, per, units, ms in (("K1 pyramid", pyr, frames, c[0]), ("K2-K4 detect", det, ndet, c[1])):
        if ms > 0:
            gbs = per * units / (ms / 1000.0) / 1e9
            out[name] = {"alg_bytes_per_unit": per, "units": units, "ms": round(float(ms), 3),
                         "achieved_gbs": round(gbs, 1), "frac": round(gbs / hbm, 4)}
    return out


def compose_issue(spec, planes, frames, ms):
    """K8's fraction of the SM issue rate (its actual limiter): warp
    instructions per launch from the committed ncu capture, scaled per frame,
    over the measured launch time, against 4 schedulers x SMs x SM clock."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "compose_traffic.json")
    try:
        t = json.load(open(p))
        inst = t["warp_instructions"] * frames / t["frames_per_launch"]
    except (OSError, ValueError, KeyError):
        return None
    if (t["width"], t["height"], t["planes"]) != (spec.width, spec.height, planes) or not ms:
        return None
    import torch

    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    try:
        import pynvml

        pynvml.nvmlInit()
        mhz = pynvml.nvmlDeviceGetMaxClockInfo(pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device()),
                                               pynvml.NVML_CLOCK_SM)
    except Exception:
        mhz = 1965
    peak = props.multi_processor_count * 4 * mhz * 1e6
    return {"warp_instructions": inst, "peak_warp_inst_per_s": peak, "frac": inst / (ms / 1000.0) / peak,
            "source": "ncu smsp__inst_executed.sum (profiles/compose_traffic.json)"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def render(cfg, first, count, pinned=False, threads=0):
    import torch

    from paper_1701_03572_b200.synth import Video

    spec = cfg.video
    v = Video(spec, threads=threads)
    planes = 3 if spec.color else 1
    shape = (count, spec.height, spec.width)
    bufs = [torch.empty(shape, dtype=torch.uint8, pin_memory=pinned) for _ in range(planes)]
    step = 50
    for f0 in range(0, count, step):
        n = min(step, count - f0)
        v.render(first + f0, n, out=[b[f0:f0 + n] for b in bufs])
    return bufs


# --------------------------------------------------------------- reference ---
def cpu_reference(cfg, frames_y, frames_cb, frames_cr, threads):
    """The reference CPU path on `threads` host threads over the given frames;
    returns frames/s."""
    import ctypes as C

    sys.path.insert(0, ROOT)
    from tests import _oracle

    ref = _oracle.reference()
    y = np.ascontiguousarray(frames_y)
    cb = None if frames_cb is None else np.ascontiguousarray(frames_cb)
    cr = None if frames_cr is None else np.ascontiguousarray(frames_cr)
    t0 = time.perf_counter()
    out = ref.stabilize_sequence(y, cfg.stab, cb, cr, compose=True, threads=threads)
    dt = time.perf_counter() - t0
    del C
    return len(y) / dt, dt, out


def sample_parity(cfg, planes, ref_out):
    """Our Stage I on the cpu_baseline sample against the reference's output
    for it (tests/_parity.py: records, parameters, pixels)."""
    from paper_1701_03572_b200 import pipeline
    from tests import _parity

    y, cb, cr = planes[0], planes[1], planes[2]
    gy, gb, gr, grec = pipeline.stabilize_sequence(y, cfg.stab, cb, cr)
    oy, ob, orr, orec = ref_out
    s = _parity.summarize(grec, orec, [gy, gb, gr], [oy, ob, orr])
    s["checker"] = "reference (oracle/_ref, unmodified sources)"
    return s


def run_reference_arm(args, cfg):
    import torch.distributed as dist  # noqa: F401

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n_total = cfg.video.frames
    # five segments per thread (the segment-parallel driver needs a few per
    # thread to keep every core busy), at most 400 frames per step
    sample = int(min(n_total, max(5 * threads * cfg.stab.flow.redetect_interval, 60)))
    sample = min(sample, 400)
    planes = render(cfg, 0, sample, pinned=False)
    arrs = [p.numpy() for p in planes] + [None] * (3 - len(planes))
    for _ in range(args.warmup):
        cpu_reference(cfg, arrs[0][: min(sample, 2 * cfg.stab.flow.redetect_interval + 1)], *[
            None if a is None else a[: min(sample, 2 * cfg.stab.flow.redetect_interval + 1)]
            for a in arrs[1:]], threads)
    times = []
    for _ in range(args.steps):
        fps, dt, _ = cpu_reference(cfg, arrs[0], arrs[1], arrs[2], threads)
        times.append(dt)
    ms = 1000.0 * float(np.mean(times))
    value = sample / (ms / 1000.0)
    desc = f"first {sample} of {n_total} frames of {args.config}, reference stage functions on {threads} threads"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE generator)",
            "config": workload(args, cfg), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload(args, cfg):
    v = cfg.video
    s = cfg.stab
    return {"workload": f"BASELINE {args.config}: {cfg.name}", "width": v.width, "height": v.height,
            "frames": v.frames, "planes": 3 if v.color else 1, "max_corners": s.detect.max_corners,
            "min_distance": s.detect.min_distance, "levels": s.flow.max_levels,
            "lk_window": 2 * s.flow.window_radius + 1, "ransac_iters": s.ransac.iterations,
            "smooth_radius": s.smooth_radius, "model": "similarity" if s.selector.mode == 2 else
            ("rigid" if s.selector.mode == 1 else "hybrid"),
            "parallelism": f"frame-shards x{args.gpus}" if args.gpus > 1 else "1 GPU",
            "l2": "inputs per step (6.2 GB at 1080p RGB) >> 126 MB L2; no flush needed",
            "seed": hex(v.seed)}


# --------------------------------------------------------------------- ours ---
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1701_03572_b200 import _lib, pipeline

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dist_backend == "gloo":  # functional check of the N > 1 path on fewer GPUs (not a measurement)
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    n = cfg.video.frames
    spec = cfg.video
    planes = 3 if spec.color else 1
    shards = pipeline.shard_ranges(n, cfg.stab.flow.redetect_interval, world)
    sh = shards[rank]
    lo, hi = sh.frames_needed if world > 1 else (0, n)
    count = hi - lo
    t0 = time.time()
    host = render(cfg, lo, count, pinned=True)
    gen_s = time.time() - t0
    dev = [h.cuda() for h in host]
    own = (sh.own_end - sh.own_begin) if world > 1 else n
    outs = [torch.empty((own,) + tuple(d.shape[1:]), dtype=d.dtype, device=d.device) for d in dev]
    host_out = [torch.empty((own,) + tuple(h.shape[1:]), dtype=h.dtype, pin_memory=True) for h in host]
    ctx = _lib.context(local)
    ctx.enable_timing(True)
    stream = torch.cuda.current_stream(local)
    ctx.set_stream(stream.cuda_stream)
    nccl = world > 1 and args.dist_backend == "nccl"
    if nccl:  # the context's own NCCL communicator: records all-gathered device to device
        pipeline.init_comm(ctx)

    chroma = (dev[1], dev[2]) if planes == 3 else (None, None)
    ochroma = (outs[1], outs[2]) if planes == 3 else (None, None)

    def step_device():
        if world == 1:
            pipeline.stabilize_sequence_device(dev[0], cfg.stab, *chroma, out_y=outs[0], out_cb=ochroma[0],
                                               out_cr=ochroma[1], records=False)
        elif nccl:
            pipeline.stabilize_sharded_device(ctx, n, dev[0], cfg.stab, *chroma, outs[0], *ochroma, records=False)
        else:  # gloo functional check: host-side exchange of the records
            pipeline.stabilize_sharded(n, dev[0], lo, cfg.stab, rank, world, *chroma, device=local)

    cfg_c = cfg.stab.c()
    rec = np.zeros(n, pipeline.RECORD_DT)

    def step_e2e():
        if world == 1:
            pipeline.stabilize_sequence_host_buffers(
                ctx, host[0], host[1] if planes == 3 else None, host[2] if planes == 3 else None,
                n, spec.width, spec.height, spec.width if planes == 3 else 0,
                spec.height if planes == 3 else 0, cfg_c, host_out[0],
                host_out[1] if planes == 3 else None, host_out[2] if planes == 3 else None, rec)
        elif nccl:  # C-ABI host-buffer entry point: chunked upload/motion, NCCL all-gather, compose/download
            pipeline.stabilize_sharded_host(ctx, n, host[0], cfg.stab, *(host[1:] if planes == 3 else (None, None)),
                                            host_out[0], *(host_out[1:] if planes == 3 else (None, None)),
                                            records=False)
        else:  # gloo: the same entry point split at the exchange
            hch = host[1:] if planes == 3 else (None, None)
            mine = pipeline.shard_motion(ctx, n, world, rank, host[0], cfg.stab, *hch)
            shards = pipeline.shard_ranges(n, cfg.stab.flow.redetect_interval, world)
            gathered = pipeline.exchange_motion(mine, max(s.count for s in shards))
            motion = pipeline.assemble_motion(n, list(zip(shards, gathered)))
            pipeline.shard_compose(ctx, n, world, rank, motion, cfg.stab, spec.width, spec.height,
                                   spec.width if planes == 3 else 0, spec.height if planes == 3 else 0,
                                   host_out[0], *(host_out[1:] if planes == 3 else (None, None)))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        barrier()
        launches0 = ctx.stats().launches
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        comp = []
        ev0.record(stream)
        for _ in range(steps):
            fn()
            s = ctx.stats()
            comp.append((s.ms_pyramid, s.ms_detect, s.ms_track, s.ms_fit, s.ms_plan, s.ms_compose))
        ev1.record(stream)
        barrier()
        ms = ev0.elapsed_time(ev1) / steps
        if world > 1:
            t = torch.tensor([ms], device="cuda" if args.dist_backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        launches = (ctx.stats().launches - launches0) // max(steps, 1)
        return ms, launches, comp

    # stage timing records event pairs on the launching stream and is read
    # after each step (no host sync inside a call), so it runs in the timed
    # region; a short pass without it checks that it costs nothing
    with ClockSampler(local) as clk:
        ms_dev, launches, comp = timed(step_device, args.steps, args.warmup)
    ctx.enable_timing(False)
    ms_dev_plain, _, _ = timed(step_device, max(1, min(args.steps, 3)), 0)
    ms_e2e, _, _ = timed(step_e2e, args.steps, args.warmup)
    ms_rgb = None
    if world == 1 and planes == 3:
        # C3 is an RGB workload: the same step from interleaved RGB host frames
        # to interleaved RGB host frames (media_io's conversions on the device:
        # per-chunk RGB -> Y/Cb/Cr after upload, Y/Cb/Cr -> RGB fused into K8's
        # store); the RGB source is the device conversion of the planes
        from paper_1701_03572_b200 import evaluate
        rgb_in = torch.empty((n, spec.height, spec.width, 3), dtype=torch.uint8, pin_memory=True)
        for f0 in range(0, n, 100):
            rgb_in[f0:f0 + 100].copy_(evaluate.ycbcr_to_rgb(dev[0][f0:f0 + 100], dev[1][f0:f0 + 100],
                                                             dev[2][f0:f0 + 100]))
        rgb_out = torch.empty_like(rgb_in).pin_memory()

        def step_rgb():
            pipeline.stabilize_sequence_rgb_host_buffers(ctx, rgb_in, n, spec.width, spec.height, cfg_c, rgb_out, rec)

        ms_rgb, _, _ = timed(step_rgb, args.steps, args.warmup)
        del rgb_in, rgb_out
    ctx.enable_timing(True)
    value = n / (ms_dev / 1000.0)
    e2e = n / (ms_e2e / 1000.0)
    fb = spec.width * spec.height * planes

    line = None
    if rank == 0:
        hbm, peak_src = peaks()
        # per-stage times of this rank (rank 0 when sharded)
        c = np.array(comp).mean(axis=0) if comp else np.zeros(6)
        # dominant HBM-bound kernel family: K8 compose (luma warp+crop and chroma),
        # algorithmic bytes = one read + one write of every plane of every frame
        alg = 2.0 * fb * (sh.own_end - sh.own_begin if world > 1 else n)
        comp_ms = float(c[5]) if c[5] > 0 else None
        achieved = alg / (comp_ms / 1000.0) / 1e9 if comp_ms else None
        stages = dict(zip(["pyramid", "detect", "track", "fit", "plan", "compose"],
                          [round(float(x), 3) for x in c]))
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_dev, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded BASELINE generator, host C)",
                "config": workload(args, cfg),
                "e2e": {"value": e2e, "unit": UNIT,
                        "h2d_bytes_per_step": fb * (sum(s.count + 1 for s in shards if s.count) if world > 1 else n),
                        "d2h_bytes_per_step": fb * n + (n * pipeline.RECORD_BYTES if world == 1 else 0),
                        "ms_per_step": ms_e2e, "steps": args.steps, "warmup": args.warmup},
                "ms_per_step_without_stage_events": ms_dev_plain,
                "e2e_rgb": None if ms_rgb is None else {
                    "value": n / (ms_rgb / 1000.0), "unit": UNIT, "h2d_bytes_per_step": fb * n,
                    "d2h_bytes_per_step": fb * n + n * pipeline.RECORD_BYTES, "ms_per_step": ms_rgb,
                    "path": "stabgpu_stabilize_sequence_rgb: interleaved RGB pinned host frames in and out"},
                "roofline": {"bound": "hbm", "kernel": "K8 compose_tma_kernel (fused warp + crop/resize, all planes)",
                             "achieved": achieved, "peak": hbm, "unit": "GB/s",
                             "frac": (achieved / hbm) if achieved else None,
                             "traffic": compose_traffic(spec, planes, sh.own_end - sh.own_begin if world > 1 else n),
                             "peak_source": peak_src,
                             "alg_bytes_per_launch": alg, "ms_per_launch": comp_ms,
                             "issue": compose_issue(spec, planes, sh.own_end - sh.own_begin if world > 1 else n,
                                                    comp_ms)},
                "kernels": kernel_rooflines(spec, cfg.stab, n if world == 1 else count, c, hbm),
                "stage_ms": stages,
                "gpu_launches": int(launches),
                "lk": {"iterations": int(ctx.stats().lk_iterations),
                       "level_builds": int(ctx.stats().lk_level_builds)},
                "clocks": clk.summary(),
                "input_gen_s": round(gen_s, 1)}
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            sample = min(n, max(6 * threads, 40))
            hs = [h[:sample].numpy() for h in host] + [None] * (3 - planes)
            fps, dt, ref_out = cpu_reference(cfg, hs[0], hs[1], hs[2], threads)
            if dt < 5.0 and sample < n:  # a short sample: take one worth ~10 s of CPU work instead
                R = cfg.stab.flow.redetect_interval
                bigger = min(n, int(fps * 10.0) // R * R + 1)
                if bigger > sample:
                    sample = bigger
                    del ref_out
                    hs = [h[:sample].numpy() for h in host] + [None] * (3 - planes)
                    fps, dt, ref_out = cpu_reference(cfg, hs[0], hs[1], hs[2], threads)
            line["cpu_baseline"] = {"value": fps, "unit": UNIT, "cores": threads, "kind": "reference",
                                    "sample": f"first {sample} frames of {args.config} "
                                              f"({dt:.1f} s, reference stage functions, segment-parallel)"}
            # parity of the same sample (outside the timed region): our Stage I on
            # those frames against the reference's output for them
            line["parity"] = sample_parity(cfg, hs, ref_out)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------ c5 streams ---
def run_streams(args, cfg, group=64):
    """BASELINE configs[4]: 256 independent 1280x720 streams of 240 frames,
    round-robin over ranks (no collective).  One step = every stream of this
    rank, stabilized through stabgpu_stabilize_streams_device in groups of
    `group` streams (one launch per stage per group); e2e = the same through
    the host-buffer entry point (pinned input, a reused pinned output group
    buffer, copies overlapped inside the call)."""
    import torch
    import torch.distributed as dist

    from paper_1701_03572_b200 import _lib, pipeline
    from paper_1701_03572_b200.synth import Video

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dist_backend == "gloo":  # functional check of the N > 1 path on fewer GPUs (not a measurement)
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    spec = cfg.video
    mine = pipeline.streams_of_rank(spec.streams, rank, world)
    S, F, h, w = len(mine), spec.frames, spec.height, spec.width
    t0 = time.time()
    host = torch.empty((S, F, h, w), dtype=torch.uint8, pin_memory=True)
    for i, k in enumerate(mine):
        Video(spec, stream=k).render(0, F, out=[host[i]])
    gen_s = time.time() - t0
    G = min(group, S)
    ctx = _lib.context(local)
    ctx.enable_timing(True)
    stream = torch.cuda.current_stream(local)
    ctx.set_stream(stream.cuda_stream)
    dev = host.cuda()
    dout = torch.empty((G, F, h, w), dtype=torch.uint8, device="cuda")
    hout = torch.empty((G, F, h, w), dtype=torch.uint8, pin_memory=True)
    cfg_c = cfg.stab.c()
    rec = np.zeros((G, F), pipeline.RECORD_DT)

    def step_device():
        for g0 in range(0, S, G):
            ns = min(G, S - g0)
            pipeline.stabilize_streams_device(dev[g0:g0 + ns], cfg.stab, out_y=dout[:ns], records=False)

    def step_e2e():
        for g0 in range(0, S, G):
            ns = min(G, S - g0)
            pipeline.stabilize_streams_host_buffers(ctx, host[g0:g0 + ns], None, None, ns, F, w, h, 0, 0,
                                                    cfg_c, hout[:ns], None, None, rec[:ns])

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        barrier()
        launches0 = ctx.stats().launches
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(steps):
            fn()
        ev1.record(stream)
        barrier()
        ms = ev0.elapsed_time(ev1) / steps
        if world > 1:
            t = torch.tensor([ms], device="cuda" if args.dist_backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, (ctx.stats().launches - launches0) // max(steps, 1)

    with ClockSampler(local) as clk:
        ms_dev, launches = timed(step_device, args.steps, args.warmup)
    ms_e2e, _ = timed(step_e2e, max(1, min(args.steps, 2)), 1)
    total = spec.streams * F  # frames all ranks process per step
    if rank == 0:
        st = ctx.stats()
        line = {"metric": METRIC, "value": total / (ms_dev / 1000.0), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_dev,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded BASELINE generator, host C, seed ^ stream)",
                "config": {"workload": f"BASELINE c5: {cfg.name}", "streams": spec.streams,
                           "frames_per_stream": F, "width": w, "height": h,
                           "max_corners": cfg.stab.detect.max_corners, "levels": cfg.stab.flow.max_levels,
                           "model": "rigid", "streams_per_call": G,
                           "parallelism": f"streams round-robin x{world}" if world > 1 else "1 GPU",
                           "l2": f"{S * F * w * h / 1e9:.1f} GB of input per step >> 126 MB L2",
                           "seed": hex(spec.seed)},
                "e2e": {"value": total / (ms_e2e / 1000.0), "unit": UNIT,
                        "h2d_bytes_per_step": S * F * w * h,
                        "d2h_bytes_per_step": S * F * (w * h + pipeline.RECORD_BYTES),
                        "ms_per_step": ms_e2e},
                "stage_ms_last_group": dict(zip(["pyramid", "detect", "track", "fit", "plan", "compose"],
                                                [round(float(x), 3) for x in (
                                                    st.ms_pyramid, st.ms_detect, st.ms_track, st.ms_fit,
                                                    st.ms_plan, st.ms_compose)])),
                "gpu_launches": int(launches), "clocks": clk.summary(), "input_gen_s": round(gen_s, 1)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: run the multi-rank code path on fewer GPUs than ranks (functional check only)")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--streams", type=int, default=0, help="c5: override the stream count (quick runs)")
    args = ap.parse_args()
    from paper_1701_03572_b200.synth import CONFIGS

    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        if args.config == "c5":
            raise SystemExit("--impl reference runs c1-c4 (c5 streams are c2-like sequences)")
        return run_reference_arm(args, cfg)
    if args.config == "c5":
        if args.streams:
            cfg.video.streams = args.streams
        return run_streams(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
