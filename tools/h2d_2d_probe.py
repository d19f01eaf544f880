"""Pinned host -> device: one linear cudaMemcpyAsync vs cudaMemcpy2DAsync of the same frames
(equal pitches), for 4K and 450x450 batches.  usage: python tools/h2d_2d_probe.py"""
import ctypes, time, torch
rt = ctypes.CDLL("libcudart.so.12")
for (n, h, w) in ((32, 2160, 3840), (256, 450, 450), (32, 1080, 1920)):
    src = torch.empty((n, h, w), dtype=torch.uint8).pin_memory()
    dst = torch.empty((n, h, w), dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    nb = n * h * w
    for mode in ("1d", "2d", "1d", "2d"):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(10):
            if mode == "1d":
                rc = rt.cudaMemcpyAsync(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                                        ctypes.c_size_t(nb), 1, ctypes.c_void_p(s))
            else:
                rc = rt.cudaMemcpy2DAsync(ctypes.c_void_p(dst.data_ptr()), ctypes.c_size_t(w),
                                          ctypes.c_void_p(src.data_ptr()), ctypes.c_size_t(w),
                                          ctypes.c_size_t(w), ctypes.c_size_t(n * h), 1, ctypes.c_void_p(s))
            assert rc == 0, rc
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 10
        print(f"{n}x{h}x{w} {mode}: {nb / dt / 1e9:.1f} GB/s")
