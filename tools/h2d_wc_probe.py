"""H2D bandwidth from write-combined pinned memory vs default pinned memory (537 MB):
the streaming copy kernel (4 and 8 CTAs) and a copy-engine cudaMemcpyAsync."""
import ctypes, os, sys, torch
import numpy as np
sys.path.insert(0, os.getcwd())
from cuda import cudart
from paper_1403_5337_b200 import _native as N
nbytes = 64 * 1024 * 1024 * 8
d = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = torch.cuda.current_stream().cuda_stream

def run(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9

for name, flags in (("default", cudart.cudaHostAllocDefault), ("write-combined", cudart.cudaHostAllocWriteCombined),
                    ("wc+mapped", cudart.cudaHostAllocWriteCombined | cudart.cudaHostAllocMapped)):
    err, hp = cudart.cudaHostAlloc(nbytes, flags)
    assert err == cudart.cudaError_t.cudaSuccess, err
    a = np.ctypeslib.as_array((ctypes.c_double * (nbytes // 8)).from_address(hp))
    a[:] = 1.5
    for c in (4, 8):
        try:
            bw = run(lambda: N.check(N.lib().hk_copy_h2d_streaming(ctypes.c_void_p(hp), N.ptr(d), nbytes, c, N.stream_handle())))
            print(f"{name:15s} stream kernel {c} CTAs: {bw:6.1f} GB/s")
        except Exception as ex:
            print(name, "stream kernel failed:", ex)
    bw = run(lambda: cudart.cudaMemcpyAsync(d.data_ptr(), hp, nbytes, cudart.cudaMemcpyKind.cudaMemcpyHostToDevice, st))
    print(f"{name:15s} cudaMemcpyAsync: {bw:6.1f} GB/s   check {float(d[12345]):.2f}")
    cudart.cudaFreeHost(hp)
