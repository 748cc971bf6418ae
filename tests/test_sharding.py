"""Host-side logic of the sharded Stage I (pipeline.shard_ranges,
assemble_motion, exchange_motion): partition properties, and a world-size-2
gloo run whose per-rank motion comes from the reference's own Trackers
(oracle/_ref ref_motion_chunk) and whose gathered plan must equal the
single-process reference run bit for bit."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

from paper_1701_03572_b200 import _abi, pipeline

from . import _data, _oracle


@pytest.mark.parametrize("R", [1, 2, 5, 7])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [2, 3, 6, 11, 53, 1000])
def test_shard_ranges_partition(n, R, world):
    shards = pipeline.shard_ranges(n, R, world)
    assert len(shards) == world
    motion = np.zeros(n, int)
    own = np.zeros(n, int)
    for sh in shards:
        if sh.count:
            assert sh.first % R == 0  # chunks start on re-detect frames
            motion[sh.first + 1: sh.first + sh.count + 1] += 1
        own[sh.own_begin: sh.own_end] += 1
        lo, hi = sh.frames_needed
        assert lo <= sh.first and hi >= min(sh.first + sh.count + 1, n)
    assert (motion[1:] == 1).all() and motion[0] == 0  # each frame pair fitted once
    assert (own == 1).all()  # each frame composed once


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("S", [1, 7, 256])
def test_streams_of_rank_round_robin(S, world):
    got = [pipeline.streams_of_rank(S, g, world) for g in range(world)]
    flat = sorted(k for part in got for k in part)
    assert flat == list(range(S))  # every stream on exactly one rank
    assert max(map(len, got)) - min(map(len, got)) <= 1  # balanced
    for g, part in enumerate(got):
        assert all(k % world == g for k in part)
    with pytest.raises(ValueError):
        pipeline.streams_of_rank(S, world, world)


def _ref_motion(y, first, count, cfg):
    ref = _oracle.reference()
    out = np.zeros(count + 1, pipeline.MOTION_DT)
    c = cfg.c()
    chunk = np.ascontiguousarray(y[first: first + count + 1])
    ref.check(ref.motion_chunk_raw(C.c_void_p(chunk.ctypes.data), first, count, y.shape[2],
                                   y.shape[1], C.byref(c), C.c_void_p(out.ctypes.data)))
    return out


def _ref_plan(motion, cfg):
    ref = _oracle.reference()
    rec = np.zeros(len(motion), pipeline.RECORD_DT)
    c = cfg.c()
    ref.check(ref.plan_corrections_raw(C.c_void_p(motion.ctypes.data), len(motion), C.byref(c),
                                       C.c_void_p(rec.ctypes.data)))
    return rec


needs_ref = pytest.mark.skipif(not _oracle.have_reference(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("world", [2, 3, 5])
def test_assembled_plan_equals_sequential(world):
    y = _data.video(frames=27, objects=1)[0]
    cfg = _data.small_cfg(_data.MODES["hybrid"], ransac=50)
    _, _, _, want = _oracle.reference().stabilize_sequence(y, cfg, threads=1)
    shards = pipeline.shard_ranges(len(y), cfg.flow.redetect_interval, world)
    parts = [(sh, _ref_motion(y, sh.first, sh.count, cfg)) for sh in shards if sh.count]
    got = _ref_plan(pipeline.assemble_motion(len(y), parts), cfg)
    assert got.tobytes() == want.tobytes()


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        y = _data.video(frames=33, objects=1)[0]
        cfg = _data.small_cfg(_data.MODES["similarity"], ransac=50)
        shards = pipeline.shard_ranges(len(y), cfg.flow.redetect_interval, world)
        sh = shards[rank]
        mine = _ref_motion(y, sh.first, sh.count, cfg) if sh.count else np.zeros(1, pipeline.MOTION_DT)
        gathered = pipeline.exchange_motion(mine, max(s.count for s in shards))
        rec = _ref_plan(pipeline.assemble_motion(len(y), list(zip(shards, gathered))), cfg)
        q.put((rank, rec.tobytes()))
    finally:
        dist.destroy_process_group()


@needs_ref
def test_gloo_world2_exchange():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y = _data.video(frames=33, objects=1)[0]
    cfg = _data.small_cfg(_data.MODES["similarity"], ransac=50)
    _, _, _, want = _oracle.reference().stabilize_sequence(y, cfg, threads=1)
    assert res[0] == res[1] == want.tobytes()
    assert (want["frame_kind"][1:] == _abi.FRAME_TRACKED).all()


@pytest.mark.parametrize("R", [1, 5, 7])
@pytest.mark.parametrize("world", [1, 2, 3, 8, 11])
@pytest.mark.parametrize("n", [2, 3, 11, 53, 1000])
def test_library_partition_equals_python(n, R, world):
    """stabgpu_shard_range (the C ABI's partition, host-only) == shard_ranges."""
    assert [pipeline.shard_range_c(n, R, world, g) for g in range(world)] == pipeline.shard_ranges(n, R, world)
