"""PCIe copy throughput of the e2e pipeline's copy shapes (no profiler): one
100 MB copy versus K chunks, 1-D versus the pipeline's 3-row strided 2-D copies
(cudaMemcpy2DAsync through pff_copy_components), one direction versus both at
once on two streams (python tools/pcie_chunks.py on a GPU)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_00331_b200 import _lib  # noqa: E402

L = _lib.load()
n = 4_198_401 + 1024                     # configs[1] scalar nodes
tot = 3 * n
h1 = torch.empty(tot, dtype=torch.float64).pin_memory()
h2 = torch.empty(tot, dtype=torch.float64).pin_memory()
d1 = torch.empty(tot, dtype=torch.float64, device="cuda")
d2 = torch.empty(tot, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def chunks(K):
    return [(k * n // K, (k + 1) * n // K) for k in range(K)]


def h2d(K, two_d):
    for a, b in chunks(K):
        if two_d:
            L.pff_copy_components(d1.data_ptr() + 8 * a, h1.data_ptr() + 8 * a, b - a, 3, n, s1.cuda_stream)
        else:
            for c in range(3):
                L.pff_copy_components(d1.data_ptr() + 8 * (c * n + a), h1.data_ptr() + 8 * (c * n + a),
                                      b - a, 1, b - a, s1.cuda_stream)


def d2h(K, two_d):
    for a, b in chunks(K):
        if two_d:
            L.pff_copy_components(h2.data_ptr() + 8 * a, d2.data_ptr() + 8 * a, b - a, 3, n, s2.cuda_stream)
        else:
            for c in range(3):
                L.pff_copy_components(h2.data_ptr() + 8 * (c * n + a), d2.data_ptr() + 8 * (c * n + a),
                                      b - a, 1, b - a, s2.cuda_stream)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


for K in (1, 4, 10, 30):
    for two_d in (False, True):
        a = timed(lambda: h2d(K, two_d))
        b = timed(lambda: d2h(K, two_d))
        c = timed(lambda: (h2d(K, two_d), d2h(K, two_d)))
        print(f"K={K:2d} {'2d' if two_d else '1d'}: h2d {8 * tot / a / 1e9:5.1f} GB/s, d2h "
              f"{8 * tot / b / 1e9:5.1f} GB/s, both {16 * tot / c / 1e9:5.1f} GB/s total "
              f"({c * 1e3:.2f} ms for 2 x {8 * tot / 1e6:.0f} MB)", flush=True)
