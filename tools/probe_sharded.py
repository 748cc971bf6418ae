"""Times the sharded Stage I code path (motion chunk -> NCCL all-gather ->
plan -> compose) with a one-rank NCCL group on one GPU, next to the plain
device path: the host-side overhead the multi-GPU bench adds per step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_1701_03572_b200 import pipeline, synth
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29511")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 250
cfg = synth.CONFIGS[name]
planes = [torch.from_numpy(p).cuda() for p in synth.Video(cfg.video).render(0, n)]
cb, cr = (planes[1], planes[2]) if len(planes) == 3 else (None, None)
def dev():
    pipeline.stabilize_sequence_device(planes[0], cfg.stab, cb, cr, records=False)
def shard():
    pipeline.stabilize_sharded(n, planes[0], 0, cfg.stab, 0, 1, cb, cr)
for fn in (dev, shard):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    print(f"{fn.__name__}: {(time.perf_counter() - t) / 3 * 1e3:.2f} ms for {n} frames")
dist.destroy_process_group()
