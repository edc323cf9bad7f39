"""How fast can the host output pool be page-locked?  cudaHostAlloc vs mmap + transparent huge
pages + parallel first touch + cudaHostRegister (mapped).  usage: pin_probe.py [GB]"""
import ctypes as C
import mmap
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_15964_b200 as cp  # noqa: E402
from paper_2501_15964_b200 import _lib as L  # noqa: E402

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
nbytes = int(gb * (1 << 30))
cp.default_context()
t0 = time.perf_counter()
h = C.c_void_p()
L.check(L.load().cp_host_alloc(nbytes, C.byref(h)))
t1 = time.perf_counter()
L.load().cp_host_free(h)
print(f"cudaHostAlloc {gb} GB: {t1 - t0:.2f} s", flush=True)

libc = C.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = C.c_void_p
libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
cudart = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
t0 = time.perf_counter()
p = libc.mmap(None, nbytes, mmap.PROT_READ | mmap.PROT_WRITE, mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
libc.madvise(p, nbytes, 14)  # MADV_HUGEPAGE
nth = min(32, os.cpu_count() or 8)
chunk = nbytes // nth


def touch(k):
    base = p + k * chunk
    end = nbytes if k == nth - 1 else (k + 1) * chunk
    C.memset(base, 0, end - k * chunk)


ths = [threading.Thread(target=touch, args=(k,)) for k in range(nth)]
for t in ths:
    t.start()
for t in ths:
    t.join()
t1 = time.perf_counter()
import torch  # noqa: E402
rt = torch.cuda.cudart()
r = rt.cudaHostRegister(p, nbytes, 0x01 | 0x02)  # portable | mapped
t2 = time.perf_counter()
print(f"mmap+THP+touch({nth} threads) {t1 - t0:.2f} s, cudaHostRegister {t2 - t1:.2f} s (rc {r})", flush=True)
