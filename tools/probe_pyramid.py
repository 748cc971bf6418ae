"""Times K1 (pyramid levels, Stage I batch layout) alone on device-resident frames."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
from paper_1701_03572_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
w, h = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (1920, 1080)
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(1)
src = torch.randint(0, 256, (n, h, w), dtype=torch.uint8, device="cuda", generator=g)
dims = [(w, h)]
while len(dims) < 4 and dims[-1][0] // 2 >= 16 and dims[-1][1] // 2 >= 16:
    dims.append((dims[-1][0] // 2, dims[-1][1] // 2))
lv = [src] + [torch.empty((n, hh, ww), dtype=torch.uint8, device="cuda") for ww, hh in dims[1:]]
st = torch.cuda.current_stream().cuda_stream
def run():
    for l in range(1, len(dims)):
        lib.stabgpu_debug_pyramid_level(C.c_void_p(lv[l - 1].data_ptr()), C.c_size_t(dims[l - 1][0] * dims[l - 1][1]),
                                        dims[l - 1][0], dims[l - 1][1], C.c_void_p(lv[l].data_ptr()),
                                        C.c_size_t(dims[l][0] * dims[l][1]), n, C.c_void_p(st))
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
alg = n * sum(a * b for a, b in dims)
print(f"pyramid {n}x{w}x{h} L{len(dims)}: {ms:.3f} ms  {alg / ms / 1e6:.0f} GB/s algorithmic")
