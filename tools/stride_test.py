"""Fused top-K at 4000 x 32768 with padded leading dimensions and fresh
allocations: does the row stride / placement change the achieved bandwidth?"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import time_rotating
from paper_1805_02867_b200 import _lib

lib = _lib.load()
dev = torch.device("cuda", 0)
rows, V, k = 4000, 32768, 5
vals = torch.empty((rows, k), device=dev)
idx = torch.empty((rows, k), dtype=torch.int64, device=dev)
ws = torch.zeros(4096, dtype=torch.uint8, device=dev)
junk = []
for trial in range(3):
    for pad in (0, 4, 32, 256, 1024):
        ld = V + pad
        n = 2
        x = torch.empty((n, rows, ld), device=dev).normal_()

        def launch(i, st):
            assert lib.osmx_softmax_topk(5, x[i].data_ptr(), ld, rows, V, k, vals.data_ptr(), idx.data_ptr(),
                                         ws.data_ptr(), ws.numel(), st) == 0

        ms, _ = time_rotating(launch, n, 9)
        print(f"trial {trial} pad {pad:>5}: {ms:.4f} ms  {4 * rows * V / ms / 1e6:.0f} GB/s", flush=True)
        del x
    junk.append(torch.empty(300 << 20, dtype=torch.uint8, device=dev))  # shift later allocations
