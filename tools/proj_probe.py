import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1805_02867_b200 import _lib, osmx
for kv in sys.argv[1:]:
    _lib.config_set(kv.split("=")[0], int(kv.split("=")[1]))
rows, D, V = 4096, 4096, 32768
h = (torch.randn((rows, D), device="cuda") / 8).to(torch.bfloat16)
w = (torch.randn((V, D), device="cuda") / 8).to(torch.bfloat16)
for _ in range(2):
    osmx.proj_softmax_topk(h, w, 5, check=False)
torch.cuda.synchronize()
print("ok")
