"""H2D / D2H bandwidth by host-allocation kind (the e2e leg's bound): torch pin_memory,
cudaHostAlloc default / write-combined / portable+mapped, cudaHostRegister of malloc'd memory,
pageable.  8 MiB (c2's X) and 256 MiB; CUDA events around 20 copies."""
import ctypes
import torch

rt = ctypes.CDLL("libcudart.so.12")
rt.cudaHostAlloc.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, ctypes.c_uint]
rt.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]


def host_buf(kind, nbytes):
    if kind == "torch_pinned":
        t = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        return t.data_ptr(), t
    if kind == "pageable":
        t = torch.empty(nbytes, dtype=torch.uint8)
        return t.data_ptr(), t
    if kind == "malloc+register":
        t = torch.empty(nbytes, dtype=torch.uint8)
        assert rt.cudaHostRegister(ctypes.c_void_p(t.data_ptr()), nbytes, 0) == 0
        return t.data_ptr(), t
    p = ctypes.c_void_p()
    flags = {"hostalloc_default": 0, "hostalloc_wc": 4, "hostalloc_portable_mapped": 1 | 2}[kind]
    assert rt.cudaHostAlloc(ctypes.byref(p), nbytes, flags) == 0
    return p.value, None


for nbytes in (8 << 20, 256 << 20):
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for kind in ("torch_pinned", "hostalloc_default", "hostalloc_wc", "hostalloc_portable_mapped", "malloc+register",
                 "pageable"):
        ptr, keep = host_buf(kind, nbytes)
        res = []
        for direction, kindc in (("h2d", 1), ("d2h", 2)):
            src, dst = (ptr, d.data_ptr()) if kindc == 1 else (d.data_ptr(), ptr)
            for _ in range(3):
                rt.cudaMemcpyAsync(ctypes.c_void_p(dst), ctypes.c_void_p(src), nbytes, kindc, ctypes.c_void_p(st))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                rt.cudaMemcpyAsync(ctypes.c_void_p(dst), ctypes.c_void_p(src), nbytes, kindc, ctypes.c_void_p(st))
            e1.record()
            torch.cuda.synchronize()
            res.append(f"{direction} {nbytes * 20 / e0.elapsed_time(e1) / 1e6:6.1f} GB/s")
        print(f"{nbytes >> 20:4d} MiB {kind:26s} " + "  ".join(res), flush=True)
