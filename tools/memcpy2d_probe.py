"""Cost of the (H,W,2) interleave of the v planes as two 4-byte-wide
cudaMemcpy2DAsync D2D copies vs a torch strided copy (diagnostic)."""
import ctypes as C
import torch

rt = C.CDLL("libcudart.so.12") if False else None
try:
    rt = C.CDLL("libcudart.so")
except OSError:
    import glob, os
    cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))
    cands += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    rt = C.CDLL(cands[0])
n = 1 << 20
src = torch.randn(2 * n, device="cuda")
dst = torch.empty(n, 2, device="cuda")
st = torch.cuda.current_stream().cuda_stream
def memcpy2d():
    for k in range(2):
        rc = rt.cudaMemcpy2DAsync(C.c_void_p(dst.data_ptr() + 4 * k), C.c_size_t(8),
                                  C.c_void_p(src.data_ptr() + 4 * k * n), C.c_size_t(4),
                                  C.c_size_t(4), C.c_size_t(n), C.c_int(3), C.c_void_p(st))
        assert rc == 0, rc
def tcopy():
    dst.copy_(src.view(2, n).t())
for name, f in (("memcpy2d", memcpy2d), ("torch", tcopy)):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(name, round(e0.elapsed_time(e1) / 20 * 1e3, 1), "us")

# contiguous D2D memcpy / memset of the level-start state (1024^2: 12 planes)
big_s = torch.randn(12 * n, device="cuda")
big_d = torch.empty_like(big_s)
def d2d():
    assert rt.cudaMemcpyAsync(C.c_void_p(big_d.data_ptr()), C.c_void_p(big_s.data_ptr()),
                              C.c_size_t(12 * n * 4), C.c_int(3), C.c_void_p(st)) == 0
def mset():
    assert rt.cudaMemsetAsync(C.c_void_p(big_d.data_ptr()), C.c_int(0), C.c_size_t(12 * n * 4),
                              C.c_void_p(st)) == 0
def tcopy_big():
    big_d.copy_(big_s)
for name, f in (("d2d 48MB", d2d), ("memset 48MB", mset), ("torch copy 48MB", tcopy_big)):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(name, round(e0.elapsed_time(e1) / 20 * 1e3, 1), "us")
