"""cudaHostRegister / Unregister throughput on the box (pageable staging design aid)."""
import ctypes
import time

import numpy as np
import torch

rt = ctypes.CDLL("libcudart.so.12") if False else None
torch.cuda.init()
cr = torch.cuda.cudart()
props = torch.cuda.get_device_properties(0)
lib = ctypes.CDLL(torch._C.__file__.replace("_C.cpython-312-x86_64-linux-gnu.so", "lib/libcudart.so.12"), mode=ctypes.RTLD_GLOBAL) if False else None
try:
    cudart = ctypes.CDLL("libcudart.so")
except OSError:
    import glob
    cudart = ctypes.CDLL(glob.glob("/usr/local/cuda/lib64/libcudart.so*")[0])
v = ctypes.c_int(0)
for name, attr in (("pageableMemoryAccess", 88), ("pageableMemoryAccessUsesHostPageTables", 100),
                   ("hostRegisterSupported", 99), ("directManagedMemAccessFromHost", 101)):
    cudart.cudaDeviceGetAttribute(ctypes.byref(v), attr, 0)
    print(f"{name}: {v.value}")
for mb in (64, 256, 1024, 4096):
    a = np.ones(mb << 18, np.float32)  # touched
    p = a.ctypes.data
    t0 = time.perf_counter()
    rc = cudart.cudaHostRegister(ctypes.c_void_p(p), ctypes.c_size_t(a.nbytes), 0)
    t1 = time.perf_counter()
    rc2 = cudart.cudaHostUnregister(ctypes.c_void_p(p))
    t2 = time.perf_counter()
    print(f"{mb:5d} MiB register {a.nbytes / (t1 - t0) / 1e9:7.1f} GB/s  unregister {a.nbytes / (t2 - t1) / 1e9:7.1f} GB/s rc={rc},{rc2}")
