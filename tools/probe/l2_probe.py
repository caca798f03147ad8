"""Driver of l2_probe.cu (see there): for each buffer size, pass 1 (shift 0)
then pass 2 with shift 0 (same SMs re-read their slices), then shift =
blocks / 2 (other SMs read them). Run under ncu --metrics dram__bytes_read.sum."""
import ctypes
import os
import subprocess
import sys

import torch

here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "l2_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so, os.path.join(here, "l2_probe.cu")])
lib = ctypes.CDLL(so)
lib.l2_probe.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
sink = torch.zeros(1, dtype=torch.int64, device="cuda")
blocks = 148
for mb in [int(v) for v in (sys.argv[1:] or ["32", "56", "80", "110"])]:
    buf = torch.randint(0, 255, (mb << 20,), dtype=torch.uint8, device="cuda")
    for shift in (0, 0, blocks // 2, 1):
        lib.l2_probe(buf.data_ptr(), buf.numel(), blocks, shift, sink.data_ptr())
    torch.cuda.synchronize()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    flush.fill_(1)
    del buf, flush
print("ok")
