"""Does a large resident allocation change the fused top-K time at 4000 x 32K?"""
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


def run(tag):
    x = torch.empty((2, rows, V), device=dev).normal_()

    def launch(i, st):
        assert lib.osmx_softmax_topk(5, x[i].data_ptr(), V, rows, V, k, vals.data_ptr(), idx.data_ptr(),
                                     ws.data_ptr(), ws.numel(), st) == 0

    ms, mn = time_rotating(launch, 2, 9)
    print(f"{tag:>28}: median {ms:.4f} ms  min {mn:.4f}  base {x.data_ptr():#x}", flush=True)
    del x


run("fresh")
big = torch.empty(65536 * 131072, dtype=torch.float32, device=dev)
big.normal_()
run("after 34 GB resident")
run("again")
del big
torch.cuda.empty_cache()
run("34 GB freed")
