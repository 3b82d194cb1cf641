import time, ctypes
import torch
from cuda import cudart
n, k, kb = 525825, 32, 8
elt = 16
host = torch.empty(n * k * 2, dtype=torch.float64).pin_memory()
dev_full = torch.empty(n * k * 2, dtype=torch.float64, device="cuda")
dev_g = torch.empty(n * kb * 2, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
full = lambda: cudart.cudaMemcpyAsync(dev_full.data_ptr(), host.data_ptr(), n * k * elt, cudart.cudaMemcpyKind.cudaMemcpyHostToDevice, s.cuda_stream)
g2d = lambda: cudart.cudaMemcpy2DAsync(dev_g.data_ptr(), kb * elt, host.data_ptr(), k * elt, kb * elt, n, cudart.cudaMemcpyKind.cudaMemcpyHostToDevice, s.cuda_stream)
d2h = lambda: cudart.cudaMemcpyAsync(host.data_ptr(), dev_full.data_ptr(), n * k * elt, cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost, s.cuda_stream)
g2d_d2h = lambda: cudart.cudaMemcpy2DAsync(host.data_ptr(), k * elt, dev_g.data_ptr(), kb * elt, kb * elt, n, cudart.cudaMemcpyKind.cudaMemcpyDeviceToHost, s.cuda_stream)
tf = t(full); print(f"H2D contiguous {n*k*elt/1e6:.0f} MB: {1e3*tf:.2f} ms, {n*k*elt/tf/1e9:.1f} GB/s")
tg = t(g2d); print(f"H2D 2D (width {kb*elt} B of pitch {k*elt} B) {n*kb*elt/1e6:.0f} MB: {1e3*tg:.2f} ms, {n*kb*elt/tg/1e9:.1f} GB/s")
td = t(d2h); print(f"D2H contiguous: {1e3*td:.2f} ms, {n*k*elt/td/1e9:.1f} GB/s")
tg2 = t(g2d_d2h); print(f"D2H 2D: {1e3*tg2:.2f} ms, {n*kb*elt/tg2/1e9:.1f} GB/s")
