"""One-row V = 2^26 (configs[4]) fused top-5 / online softmax launches for ncu."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1805_02867_b200 import _lib

lib = _lib.load()
for kv in sys.argv[1:]:
    _lib.config_set(kv.split("=")[0], int(kv.split("=")[1]))
dev = torch.device("cuda", 0)
V, k = 1 << 26, 5
x = torch.empty((1, V), device=dev).normal_()
y = torch.empty_like(x)
vals = torch.empty((1, k), device=dev)
idx = torch.empty((1, k), dtype=torch.int64, device=dev)
nb = max(lib.osmx_workspace_bytes(5, 1, V, k), lib.osmx_workspace_bytes(2, 1, V, 0))
ws = torch.zeros(nb, dtype=torch.uint8, device=dev)
sp = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    assert lib.osmx_softmax_topk(5, x.data_ptr(), V, 1, V, k, vals.data_ptr(), idx.data_ptr(), ws.data_ptr(), nb, sp) == 0
    assert lib.osmx_softmax(2, x.data_ptr(), V, y.data_ptr(), V, 1, V, ws.data_ptr(), nb, sp) == 0
torch.cuda.synchronize()
print("ok")
