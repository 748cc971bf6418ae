"""Stage I (whole-sequence) stabilization: the run_offline semantics of the
reference (pipeline.cpp:182-235) as batched B200 work, on one GPU or sharded
over the GPUs of one box.

Sharding: tracking state resets at every re-detect frame
(flow.cpp:326-330), so segments [sR, (s+1)R] are independent.  Rank g owns a
contiguous run of segments, needs one halo frame at its end, and produces the
motion records of its frames.  The small records (~100 B/frame) are
all-gathered (NCCL over NVLink on GPUs, gloo in the CPU tests); every rank
then runs the sequential selector/trajectory/smoothing scan on identical
input — bit-identical corrections everywhere — and composes its own frames.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._lib import InvalidConfigError, check, context, load
from .stab import StabConfig

MOTION_BYTES = C.sizeof(_abi.MotionRecord)
RECORD_BYTES = C.sizeof(_abi.FrameRecord)

# numpy views of the C records
DELTA_DT = np.dtype([("dx", "f8"), ("dy", "f8"), ("da", "f8"), ("dls", "f8"), ("kind", "i4"),
                     ("skipped", "i4")])
TRANSFORM_DT = np.dtype([("tx", "f8"), ("ty", "f8"), ("theta", "f8"), ("s", "f8"), ("kind", "i4"),
                         ("pad", "i4")])
RECORD_DT = np.dtype([("delta", DELTA_DT), ("correction", TRANSFORM_DT), ("frame_kind", "i4"),
                      ("n_tracks", "i4"), ("n_inliers", "i4"), ("decision", "i4")])
MOTION_DT = np.dtype([("rigid", DELTA_DT), ("similarity", DELTA_DT), ("e_rigid", "f8"),
                      ("e_similarity", "f8"), ("frame_kind", "i4"), ("n_tracks", "i4"),
                      ("n_inliers_rigid", "i4"), ("n_inliers_similarity", "i4"), ("status", "i4"),
                      ("pad", "i4")])
assert RECORD_DT.itemsize == RECORD_BYTES, (RECORD_DT.itemsize, RECORD_BYTES)
assert MOTION_DT.itemsize == MOTION_BYTES, (MOTION_DT.itemsize, MOTION_BYTES)


def _vp(x) -> C.c_void_p:
    """Pointer of a numpy array or torch tensor (None -> NULL)."""
    if x is None:
        return C.c_void_p(0)
    if isinstance(x, np.ndarray):
        return C.c_void_p(x.ctypes.data)
    return C.c_void_p(x.data_ptr())


# ------------------------------------------------------------- one GPU ------
def stabilize_sequence(y: np.ndarray, cfg: StabConfig, cb: np.ndarray | None = None,
                       cr: np.ndarray | None = None, device: int = 0):
    """Host planes in, host planes out (copies overlapped inside the call).

    y: (n, h, w) uint8; cb/cr: (n, ch, cw) uint8 or None.
    Returns (out_y, out_cb, out_cr, records) with records a RECORD_DT array."""
    y = np.ascontiguousarray(y, np.uint8)
    n, h, w = y.shape
    oy = np.empty_like(y)
    ocb = ocr = None
    ch = cw = 0
    if cb is not None:
        cb = np.ascontiguousarray(cb, np.uint8)
        cr = np.ascontiguousarray(cr, np.uint8)
        _, ch, cw = cb.shape
        ocb, ocr = np.empty_like(cb), np.empty_like(cr)
    rec = np.zeros(n, RECORD_DT)
    c = cfg.c()
    check(load().stabgpu_stabilize_sequence(context(device).handle, _vp(y), _vp(cb), _vp(cr), n, w,
                                            h, cw, ch, C.byref(c), _vp(oy), _vp(ocb), _vp(ocr),
                                            _vp(rec)))
    return oy, ocb, ocr, rec


def stabilize_sequence_host_buffers(ctx, y, cb, cr, n, w, h, cw, ch, cfg_c, oy, ocb, ocr, rec):
    """Raw C-ABI call on caller-owned (e.g. pinned torch) host buffers."""
    check(load().stabgpu_stabilize_sequence(ctx.handle, _vp(y), _vp(cb), _vp(cr), n, w, h, cw, ch,
                                            C.byref(cfg_c), _vp(oy), _vp(ocb), _vp(ocr), _vp(rec)))


def stabilize_sequence_rgb_host_buffers(ctx, rgb, n, w, h, cfg_c, out_rgb, rec):
    """Raw C-ABI call: interleaved RGB host frames in and out (media_io load /
    save conversions on the device around run_offline)."""
    check(load().stabgpu_stabilize_sequence_rgb(ctx.handle, _vp(rgb), n, w, h, C.byref(cfg_c), _vp(out_rgb),
                                                _vp(rec)))


def stabilize_sequence_device(y, cfg: StabConfig, cb=None, cr=None, out_y=None, out_cb=None,
                              out_cr=None, device: int | None = None, records: bool = True):
    """Device-resident planes (torch CUDA tensors) in and out."""
    import torch

    n, h, w = y.shape
    dev = y.device.index if device is None else device
    out_y = torch.empty_like(y) if out_y is None else out_y
    ch = cw = 0
    if cb is not None:
        _, ch, cw = cb.shape
        out_cb = torch.empty_like(cb) if out_cb is None else out_cb
        out_cr = torch.empty_like(cr) if out_cr is None else out_cr
    rec = np.zeros(n, RECORD_DT) if records else None
    c = cfg.c()
    ctx = context(dev)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    check(load().stabgpu_stabilize_sequence_device(ctx.handle, _vp(y), _vp(cb), _vp(cr), n, w, h,
                                                   cw, ch, C.byref(c), _vp(out_y), _vp(out_cb),
                                                   _vp(out_cr), _vp(rec)))
    return out_y, out_cb, out_cr, rec


# ------------------------------------------------------- many streams ------
def stabilize_streams(y: np.ndarray, cfg: StabConfig, cb: np.ndarray | None = None,
                      cr: np.ndarray | None = None, device: int = 0):
    """BASELINE configs[4]: S independent sequences of F frames each.

    y: (S, F, h, w) uint8; cb/cr: (S, F, ch, cw) or None.  Every stream is
    stabilized exactly as run_offline would on that stream alone; all streams
    share one launch per stage.  Returns (out_y, out_cb, out_cr, records) with
    records of shape (S, F)."""
    y = np.ascontiguousarray(y, np.uint8)
    S, F, h, w = y.shape
    oy = np.empty_like(y)
    ocb = ocr = None
    ch = cw = 0
    if cb is not None:
        cb = np.ascontiguousarray(cb, np.uint8)
        cr = np.ascontiguousarray(cr, np.uint8)
        ch, cw = cb.shape[2:]
        ocb, ocr = np.empty_like(cb), np.empty_like(cr)
    rec = np.zeros((S, F), RECORD_DT)
    c = cfg.c()
    check(load().stabgpu_stabilize_streams(context(device).handle, _vp(y), _vp(cb), _vp(cr), S, F, w,
                                           h, cw, ch, C.byref(c), _vp(oy), _vp(ocb), _vp(ocr),
                                           _vp(rec)))
    return oy, ocb, ocr, rec


def stabilize_streams_host_buffers(ctx, y, cb, cr, S, F, w, h, cw, ch, cfg_c, oy, ocb, ocr, rec):
    """Raw C-ABI call on caller-owned (e.g. pinned torch) host buffers."""
    check(load().stabgpu_stabilize_streams(ctx.handle, _vp(y), _vp(cb), _vp(cr), S, F, w, h, cw, ch,
                                           C.byref(cfg_c), _vp(oy), _vp(ocb), _vp(ocr), _vp(rec)))


def stabilize_streams_device(y, cfg: StabConfig, cb=None, cr=None, out_y=None, out_cb=None,
                             out_cr=None, device: int | None = None, records: bool = True):
    """Device-resident (S, F, h, w) torch CUDA tensors in and out."""
    import torch

    S, F, h, w = y.shape
    dev = y.device.index if device is None else device
    out_y = torch.empty_like(y) if out_y is None else out_y
    ch = cw = 0
    if cb is not None:
        ch, cw = cb.shape[2:]
        out_cb = torch.empty_like(cb) if out_cb is None else out_cb
        out_cr = torch.empty_like(cr) if out_cr is None else out_cr
    rec = np.zeros((S, F), RECORD_DT) if records else None
    c = cfg.c()
    ctx = context(dev)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    check(load().stabgpu_stabilize_streams_device(ctx.handle, _vp(y), _vp(cb), _vp(cr), S, F, w, h,
                                                  cw, ch, C.byref(c), _vp(out_y), _vp(out_cb),
                                                  _vp(out_cr), _vp(rec)))
    return out_y, out_cb, out_cr, rec


def streams_of_rank(n_streams: int, rank: int, world: int) -> list[int]:
    """Round-robin assignment of independent streams to ranks (BASELINE
    configs[4]).  Streams share nothing, so there is no collective."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(range(rank, n_streams, world))


# ------------------------------------------------------------- sharding -----
@dataclass(frozen=True)
class Shard:
    rank: int
    first: int        # first frame (a re-detect frame) of the motion chunk
    count: int        # frames first+1 .. first+count get motion records here
    own_begin: int    # frames this rank composes: [own_begin, own_end)
    own_end: int

    @property
    def frames_needed(self) -> tuple[int, int]:
        """Resident frame range [lo, hi) (motion chunk incl. halo, own frames)."""
        return min(self.first, self.own_begin), max(self.first + self.count + 1, self.own_end)


def shard_ranges(n: int, redetect_interval: int, world: int) -> list[Shard]:
    """Contiguous re-detect-aligned partition of an n-frame sequence."""
    if n < 2:
        raise ValueError("stabilization needs at least 2 frames")
    R = redetect_interval
    nseg = (n - 1 + R - 1) // R
    out = []
    for g in range(world):
        s0, s1 = nseg * g // world, nseg * (g + 1) // world
        first = min(s0 * R, n - 1)
        last = min(s1 * R, n - 1)
        own_begin = 0 if s0 == 0 else first + 1
        own_end = last + 1
        if s0 == s1:  # more ranks than segments: this rank idles
            first, last, own_begin, own_end = 0, 0, 0, 0
        out.append(Shard(g, first, last - first, own_begin, own_end))
    return out


def assemble_motion(n: int, parts: list[tuple[Shard, np.ndarray]]) -> np.ndarray:
    """Global motion array from per-rank chunks.

    Each part holds count+1 MOTION_DT records: entry 0 is frame `first`
    (the FIRST record on rank 0, a placeholder elsewhere), entries 1..count
    are frames first+1 .. first+count."""
    motion = np.zeros(n, MOTION_DT)
    seen = np.zeros(n, bool)
    for sh, rec in parts:
        if sh.count == 0 and sh.own_end == 0:
            continue
        if sh.first == 0:
            motion[0] = rec[0]
            seen[0] = True
        motion[sh.first + 1: sh.first + sh.count + 1] = rec[1: sh.count + 1]
        seen[sh.first + 1: sh.first + sh.count + 1] = True
    if not seen.all():
        raise RuntimeError(f"motion records missing for {int((~seen).sum())} frames")
    return motion


def exchange_motion(local: np.ndarray, max_count: int, group=None, device=None) -> list[np.ndarray]:
    """All-gather of per-rank motion arrays (padded to max_count+1 records).

    Uses NCCL device buffers when the process group is NCCL, else CPU."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    nbytes = (max_count + 1) * MOTION_BYTES
    buf = np.zeros(nbytes, np.uint8)
    raw = local.view(np.uint8)
    buf[: raw.size] = raw
    backend = dist.get_backend(group)
    dev = torch.device("cuda", device) if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(buf).to(dev)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    return [o.cpu().numpy().view(MOTION_DT) for o in outs]


def motion_chunk(y_chunk, first: int, count: int, cfg: StabConfig, device: int = 0) -> np.ndarray:
    """Motion records of frames first+1..first+count (device frames y_chunk
    hold frames first..first+count)."""
    import torch

    _, h, w = y_chunk.shape
    out = np.zeros(count + 1, MOTION_DT)
    c = cfg.c()
    ctx = context(device)
    ctx.set_stream(torch.cuda.current_stream(device).cuda_stream)
    check(load().stabgpu_motion_chunk(ctx.handle, _vp(y_chunk), first, count, w, h, C.byref(c),
                                      _vp(out)))
    return out


def plan_corrections(motion: np.ndarray, cfg: StabConfig, device: int = 0) -> np.ndarray:
    rec = np.zeros(len(motion), RECORD_DT)
    c = cfg.c()
    check(load().stabgpu_plan_corrections(context(device).handle, _vp(motion), len(motion),
                                          C.byref(c), _vp(rec)))
    return rec


def compose_frames(y, corrections: np.ndarray, crop_ratio: float, cb=None, cr=None, out_y=None,
                   out_cb=None, out_cr=None, device: int = 0):
    import torch

    n, h, w = y.shape
    ch = cw = 0
    if cb is not None:
        _, ch, cw = cb.shape
    corr = np.ascontiguousarray(corrections, TRANSFORM_DT)
    out_y = torch.empty_like(y) if out_y is None else out_y
    if cb is not None:
        out_cb = torch.empty_like(cb) if out_cb is None else out_cb
        out_cr = torch.empty_like(cr) if out_cr is None else out_cr
    ctx = context(device)
    ctx.set_stream(torch.cuda.current_stream(device).cuda_stream)
    check(load().stabgpu_compose_frames(ctx.handle, _vp(y), _vp(cb), _vp(cr), n, w, h, cw, ch,
                                        _vp(corr), crop_ratio, _vp(out_y), _vp(out_cb),
                                        _vp(out_cr)))
    return out_y, out_cb, out_cr


def stabilize_sharded(n: int, local_y, local_first: int, cfg: StabConfig, rank: int, world: int,
                      local_cb=None, local_cr=None, group=None, device: int = 0):
    """One rank of the sharded Stage I.  local_* hold frames
    [local_first, local_first + len) covering shard.frames_needed.
    Returns (out_y, out_cb, out_cr, records) for the rank's own frames."""
    shards = shard_ranges(n, cfg.flow.redetect_interval, world)
    sh = shards[rank]
    max_count = max(s.count for s in shards)
    if sh.count > 0:
        lo = sh.first - local_first
        mine = motion_chunk(local_y[lo: lo + sh.count + 1], sh.first, sh.count, cfg, device)
    else:
        mine = np.zeros(1, MOTION_DT)
    gathered = exchange_motion(mine, max_count, group, device)
    motion = assemble_motion(n, [(s, g) for s, g in zip(shards, gathered)])
    rec = plan_corrections(motion, cfg, device)
    a, b = sh.own_begin - local_first, sh.own_end - local_first
    if b <= a:
        return None, None, None, rec
    corr = rec["correction"][sh.own_begin: sh.own_end]
    oy, ob, orr = compose_frames(local_y[a:b], corr, cfg.crop_ratio,
                                 None if local_cb is None else local_cb[a:b],
                                 None if local_cr is None else local_cr[a:b], device=device)
    return oy, ob, orr, rec


def shard_range_c(n: int, redetect_interval: int, world: int, rank: int) -> Shard:
    """The library's partition (stabgpu_shard_range); equals shard_ranges()."""
    first, own_b, own_e = C.c_int64(), C.c_int64(), C.c_int64()
    count = C.c_int()
    check(load().stabgpu_shard_range(n, redetect_interval, world, rank, C.byref(first), C.byref(count),
                                     C.byref(own_b), C.byref(own_e)))
    return Shard(rank, first.value, count.value, own_b.value, own_e.value)


def init_comm(ctx, group=None) -> None:
    """Gives the context an NCCL communicator over the ranks of a
    torch.distributed group (rank 0 makes the unique id; the group broadcasts
    the 128 bytes: plumbing only, the records themselves go device to device)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = np.zeros(128, np.uint8)
    if rank == 0:
        check(load().stabgpu_nccl_unique_id(_vp(uid)))
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(uid).to(dev)
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    uid = t.cpu().numpy()
    check(load().stabgpu_comm_init(ctx.handle, _vp(uid), world, rank))


def stabilize_sharded_host(ctx, n: int, y, cfg: StabConfig, cb=None, cr=None, out_y=None, out_cb=None,
                           out_cr=None, records: bool = True):
    """One rank of the sharded Stage I through the C ABI host-buffer entry
    point (stabgpu_stabilize_sharded): y/cb/cr hold this rank's frames
    first..first+count (host, ideally pinned), out_* receive its own frames.
    The context's communicator (init_comm) sets world and rank; without one it
    is world 1."""
    _, h, w = y.shape
    ch = cw = 0
    if cb is not None:
        _, ch, cw = cb.shape
    rec = np.zeros(n, RECORD_DT) if records else None
    c = cfg.c()
    check(load().stabgpu_stabilize_sharded(ctx.handle, _vp(y), _vp(cb), _vp(cr), n, w, h, cw, ch, C.byref(c),
                                           _vp(out_y), _vp(out_cb), _vp(out_cr), _vp(rec)))
    return rec


def stabilize_sharded_device(ctx, n: int, y, cfg: StabConfig, cb=None, cr=None, out_y=None, out_cb=None,
                             out_cr=None, records: bool = True):
    """Device-resident variant (stabgpu_stabilize_sharded_device)."""
    _, h, w = y.shape
    ch = cw = 0
    if cb is not None:
        _, ch, cw = cb.shape
    rec = np.zeros(n, RECORD_DT) if records else None
    c = cfg.c()
    check(load().stabgpu_stabilize_sharded_device(ctx.handle, _vp(y), _vp(cb), _vp(cr), n, w, h, cw, ch,
                                                  C.byref(c), _vp(out_y), _vp(out_cb), _vp(out_cr), _vp(rec)))
    return rec


def shard_motion(ctx, n: int, world: int, rank: int, y, cfg: StabConfig, cb=None, cr=None) -> np.ndarray:
    """First half of stabgpu_stabilize_sharded (host-side exchange): uploads
    the rank's frames (kept resident in ctx) and returns its count+1 motion
    records."""
    sh = shard_range_c(n, cfg.flow.redetect_interval, world, rank)
    _, h, w = y.shape
    ch = cw = 0
    if cb is not None:
        _, ch, cw = cb.shape
    out = np.zeros(max(sh.count + 1, 1), MOTION_DT)
    c = cfg.c()
    check(load().stabgpu_shard_motion(ctx.handle, _vp(y), _vp(cb), _vp(cr), n, world, rank, w, h, cw, ch,
                                      C.byref(c), _vp(out)))
    return out


def shard_compose(ctx, n: int, world: int, rank: int, motion_all: np.ndarray, cfg: StabConfig, w: int, h: int,
                  cw: int = 0, ch: int = 0, out_y=None, out_cb=None, out_cr=None) -> np.ndarray:
    """Second half: plan all n frames from the gathered records and compose
    the rank's own frames from its resident ones."""
    rec = np.zeros(n, RECORD_DT)
    c = cfg.c()
    m = np.ascontiguousarray(motion_all, MOTION_DT)
    check(load().stabgpu_shard_compose(ctx.handle, _vp(m), n, world, rank, w, h, cw, ch, C.byref(c),
                                       _vp(out_y), _vp(out_cb), _vp(out_cr), _vp(rec)))
    return rec


# ------------------------------------------------------------ Stage II -----
class StreamStabilizer:
    """Stage II (one frame at a time): the reference's run_offline /
    run_streaming loop (pipeline.cpp:182-365) over the C ABI stream object.

    push() estimates the new frame's motion and returns the frames whose
    corrections became releasable (CompensationPlanner rule: none before 2r
    estimates, then every frame whose smoothing window is complete); finish()
    releases the rest.  Each released frame is (index, y, cb, cr, record) and
    is bit-identical to Stage I's output for that frame."""

    def __init__(self, cfg: StabConfig, w: int, h: int, cw: int = 0, ch: int = 0, device: int = 0,
                 graphs: bool = True, overlap_pops: bool = False, async_push: bool = False, depth: int = 1):
        # overlap_pops: push() queues the downloads of the frames released by
        # the PREVIOUS push (stabgpu_stream_pop_async), uploads and estimates
        # the new frame, then waits for them - the D2H of frame k-r overlaps
        # the H2D of frame k+1; frames come back one push late, same bytes
        self.overlap_pops = overlap_pops
        # depth (with overlap_pops): the frames popped at push k are those
        # released by push k - depth.  With a few frames in flight the device
        # runs ahead of the host: the re-detections (which start as soon as
        # their frame has landed) overlap earlier frames' K5 steps.  depth must
        # stay below the output ring (2 * smooth_radius + 2 released frames)
        if depth < 1 or (overlap_pops and depth > max(1, 2 * cfg.smooth_radius)):
            raise InvalidConfigError("StreamStabilizer: depth must lie in [1, 2 * smooth_radius]")
        self.depth = depth
        self._owed_q = []
        # async_push: push() returns before the frame's upload has landed
        # (stabgpu_stream_push_async); the stabilizer keeps the frame's arrays
        # alive and waits for the upload at the start of the next push, so with
        # a new array per frame the upload of frame k+1 overlaps the motion of k
        self.async_push = async_push
        self._held = None
        self.w, self.h, self.cw, self.ch = w, h, cw, ch
        self._c = cfg.c()
        self._lib = load()
        self._ctx = context(device)
        self._h = C.c_void_p()
        check(self._lib.stabgpu_stream_create(self._ctx.handle, C.byref(self._c), w, h, cw, ch,
                                              C.byref(self._h)))
        # per-frame CUDA graphs (default) or one launch per kernel; same results
        check(self._lib.stabgpu_stream_set_graphs(self._h, int(graphs)))

    def _pop_all(self, n: int, wait: bool = True):
        out = []
        pop = self._lib.stabgpu_stream_pop if wait else self._lib.stabgpu_stream_pop_async
        for _ in range(n):
            idx = C.c_int64()
            y = np.empty((self.h, self.w), np.uint8)
            cb = cr = None
            if self.cw:
                cb = np.empty((self.ch, self.cw), np.uint8)
                cr = np.empty((self.ch, self.cw), np.uint8)
            rec = np.zeros(1, RECORD_DT)
            check(pop(self._h, C.byref(idx), _vp(y), _vp(cb), _vp(cr), _vp(rec)))
            out.append([idx.value, y, cb, cr, rec])
        return out

    @staticmethod
    def _frames(popped):
        return [(i, y, cb, cr, rec[0]) for i, y, cb, cr, rec in popped]

    def push(self, y: np.ndarray, cb: np.ndarray | None = None, cr: np.ndarray | None = None):
        y = np.ascontiguousarray(y, np.uint8)
        cb = None if cb is None else np.ascontiguousarray(cb, np.uint8)
        cr = None if cr is None else np.ascontiguousarray(cr, np.uint8)
        n = C.c_int()
        push = self._lib.stabgpu_stream_push
        if self.async_push:
            check(self._lib.stabgpu_stream_wait_inputs(self._h))  # the previous frame's arrays may go now
            self._held = (y, cb, cr)
            push = self._lib.stabgpu_stream_push_async
        if self.overlap_pops:
            late = self._pop_all(self._owed_q.pop(0), wait=False) if len(self._owed_q) >= self.depth else []
            check(push(self._h, _vp(y), _vp(cb), _vp(cr), C.byref(n)))
            check(self._lib.stabgpu_stream_wait_pops(self._h))
            self._owed_q.append(n.value - sum(self._owed_q))  # released by this push
            return self._frames(late)
        check(push(self._h, _vp(y), _vp(cb), _vp(cr), C.byref(n)))
        return self._frames(self._pop_all(n.value))

    def finish(self):
        n = C.c_int()
        if self.async_push:
            check(self._lib.stabgpu_stream_wait_inputs(self._h))
            self._held = None
        check(self._lib.stabgpu_stream_finish(self._h, C.byref(n)))
        self._owed_q = []
        return self._frames(self._pop_all(n.value))

    def close(self):
        if self._h:
            self._lib.stabgpu_stream_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
