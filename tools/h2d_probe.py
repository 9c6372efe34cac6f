"""H2D bandwidth probe for the end-to-end path: the streaming copy kernel at
several CTA counts vs a copy-engine cudaMemcpyAsync, 537 MB pinned (64 fronts)."""
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_1403_5337_b200 import _native as N
nbytes = 64 * 1024 * 1024 * 8
h = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
h.normal_()
d = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def run(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
for c in (2, 4, 8, 16, 32):
    bw = run(lambda: N.check(N.lib().hk_copy_h2d_streaming(N.C.c_void_p(h.data_ptr()), N.ptr(d), nbytes, c, N.stream_handle())))
    print(f"stream kernel {c:3d} CTAs: {bw:6.1f} GB/s")
print(f"cudaMemcpyAsync: {run(lambda: d.copy_(h, non_blocking=True)):6.1f} GB/s")
