"""Fused top-K time on rows where selection events never happen after the
first batch (descending rows) vs standard-normal rows: the difference is
the cost of the insertion path."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import n_rotating_sets, time_rotating
from paper_1805_02867_b200 import _lib

lib = _lib.load()
dev = torch.device("cuda", 0)
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
for kv in sys.argv[1:]:
    _lib.config_set(kv.split("=")[0], int(kv.split("=")[1]))
for V in (32768, 131072):
    rows, k = 4000, 5
    n = n_rotating_sets(4 * rows * V, l2)
    for name in ("normal", "descending", "constant"):
        if name == "normal":
            x = torch.empty((n, rows, V), device=dev).normal_()
        elif name == "descending":
            x = (-torch.arange(V, device=dev, dtype=torch.float32) * 1e-4).expand(n, rows, V).contiguous()
        else:
            x = torch.zeros((n, rows, V), device=dev)
        vals = torch.empty((rows, k), device=dev)
        idx = torch.empty((rows, k), dtype=torch.int64, device=dev)
        ws = torch.zeros(4096, dtype=torch.uint8, device=dev)

        def launch(i, st):
            assert lib.osmx_softmax_topk(5, x[i].data_ptr(), V, rows, V, k, vals.data_ptr(), idx.data_ptr(),
                                         ws.data_ptr(), ws.numel(), st) == 0

        ms, _ = time_rotating(launch, n, 7)
        print(f"V={V} {name:>10}: {ms:.4f} ms  {4 * rows * V / ms / 1e6:.0f} GB/s", flush=True)
        del x
