import ctypes, os, sys
import torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpcie_gather.so"))
lib.run_gather.restype = ctypes.c_float
lib.run_gather.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
n = 1 << 28   # 1 GiB of floats in pinned host memory
src = torch.empty(n, dtype=torch.float32).pin_memory()
src.fill_(1.0)
useful = {0: 32, 1: 32, 2: 128, 3: 512}   # bytes each request unit brings (sector / line / block)
for mode in (0, 1, 2, 3):
    for blocks, threads in ((148 * 4, 256), (148 * 16, 256)):
        iters = 64
        ms = lib.run_gather(src.data_ptr(), n, mode, blocks, threads, iters)
        units = blocks * threads * iters if mode < 2 else blocks * threads // 32 * iters
        print(f"mode {mode} grid {blocks}x{threads}: {units * useful[mode] / ms / 1e6:.1f} GB/s of touched sectors/lines "
              f"({units / ms / 1e3:.1f} M requests/s)", flush=True)
