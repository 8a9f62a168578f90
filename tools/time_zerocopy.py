"""Zero-copy PCIe bandwidth from SM loads/stores vs DMA copies (tools/ only).
    python tools/time_zerocopy.py   (needs build_variants/zc_probe.cubin: nvcc -cubin tools/zc_probe.cu)"""
import ctypes
import os
import sys

import torch
from cuda.bindings import driver as cu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
torch.cuda.init()
torch.empty(1, device="cuda")
err, mod = cu.cuModuleLoad(os.path.join(ROOT, "build_variants", "zc_probe.cubin").encode())
assert err == 0, err
err, fn = cu.cuModuleGetFunction(mod, b"zc")
assert err == 0, err
nbytes = 256 << 20
hin = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
hout = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
din = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dout = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
n = nbytes // 16
sms = torch.cuda.get_device_properties(0).multi_processor_count


def launch(mode, blocks, threads=256):
    args = [ctypes.c_void_p(hin.data_ptr()), ctypes.c_void_p(hout.data_ptr()), ctypes.c_void_p(din.data_ptr()),
            ctypes.c_void_p(dout.data_ptr()), ctypes.c_long(n), ctypes.c_int(mode)]
    ptrs = (ctypes.c_void_p * len(args))(*[ctypes.addressof(a) for a in args])
    s = torch.cuda.current_stream().cuda_stream
    err, = cu.cuLaunchKernel(fn, blocks, 1, 1, threads, 1, 1, 0, s, ptrs, 0)
    assert err == 0, err


def timed(f, reps=5):
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for blocks in (sms, 2 * sms, 4 * sms, 8 * sms):
    for mode, name in ((1, "host->dev (SM loads)"), (2, "dev->host (SM stores)"), (3, "both")):
        ms = timed(lambda: launch(mode, blocks))
        print(f"blocks {blocks:5d} {name:22s}: {ms:.2f} ms = {nbytes / ms / 1e6:.1f} GB/s per direction")
print(f"DMA H2D: {nbytes / timed(lambda: din.copy_(hin, non_blocking=True)) / 1e6:.1f} GB/s")
print(f"DMA D2H: {nbytes / timed(lambda: hout.copy_(dout, non_blocking=True)) / 1e6:.1f} GB/s")
