"""Time bddc_dense_potrf (blocked 8x8 tile Cholesky + inverse) in isolation."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_07289_b200 import _capi

lib = _capi.load()
for n, count in ((64, 1), (64, 148), (64, 4096), (128, 4096), (1024, 1)):
    ld = n
    M = torch.randn(count, n, n, dtype=torch.float64, device="cuda")
    A = (M @ M.transpose(1, 2) + n * torch.eye(n, dtype=torch.float64, device="cuda")).contiguous()
    info = np.zeros(count, dtype=np.int32)
    B = A.clone()
    lib.bddc_dense_potrf(C.c_void_p(B.data_ptr()), n, ld, ld * ld, count, None, None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    ts = []
    for _ in range(reps):
        B.copy_(A)
        torch.cuda.synchronize()
        e0.record()
        lib.bddc_dense_potrf(C.c_void_p(B.data_ptr()), n, ld, ld * ld, count, None, None)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    L = torch.linalg.cholesky(A)
    err = (torch.tril(B.transpose(1, 2)) - L).abs().max().item() if n <= 128 else float("nan")
    print(f"potrf n={n:5d} count={count:5d}: {min(ts)*1e3:9.1f} us  err {err:.1e}")
