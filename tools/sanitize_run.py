"""Small launches of every kernel family (for compute-sanitizer runs)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1805_02867_b200 import _lib, osmx

_lib.load()
rng = np.random.default_rng(3)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


cases = [
    ("resident", {"shape": 1}, [(7, 100), (5, 1023), (3, 2045)]),
    ("staged", {"shape": 4}, [(300, 3001), (40, 16383)]),
    ("cluster", {"shape": 5, "cluster_size": 4}, [(40, 70001), (9, 5)]),
    ("cluster9", {"shape": 5, "cluster_size": 9}, [(20, 150001)]),
    ("cluster_auto", {"shape": 5}, [(20, 100001)]),
    ("stream", {"shape": 2}, [(3, 40001)]),
    ("split", {"shape": 3, "split_chunk": 4096}, [(2, 50001)]),
]
for name, knobs, shapes in cases:
    for kk, vv in knobs.items():
        _lib.config_set(kk, vv)
    for rows, V in shapes:
        big = rng.standard_normal((rows, V + 3)).astype(np.float32)
        xt = dev(big)[:, 1:V + 1]  # misaligned, ld = V + 3
        for alg in ("naive", "safe", "online"):
            osmx.softmax(xt, alg=alg)
        for alg in ("online_fused", "safe_fused", "safe_unfused", "online_unfused"):
            osmx.softmax_topk(xt, min(5, V), alg=alg)
        osmx.topk(xt, min(3, V))
    for kk in knobs:
        _lib.config_set(kk, 0)
for knobs in ({"topk_threads": 32, "topk_u8": 1}, {"topk_threads": 32, "topk_pipe": 1}, {"tma": 2},
              {"topk_threads": 32, "l2_prefetch": 1}):
    for kk, vv in knobs.items():
        _lib.config_set(kk, vv)
    x = dev(rng.standard_normal((64, 20001)).astype(np.float32))
    osmx.softmax_topk(x, 5)
    osmx.topk(x, 7)
    for kk in knobs:
        _lib.config_set(kk, -1 if kk in ("topk_u8", "l2_prefetch") else 0)
x = dev(rng.standard_normal((3, 5000)).astype(np.float32))
osmx.softmax_topk(x, 100)  # large k
osmx.topk(x, 5000)
x = dev(rng.standard_normal((4, 20011)).astype(np.float32))
osmx.softmax_topk(x, 1000)  # large k: two-pass shared-memory path with the candidate trim
osmx.softmax_topk(dev(np.ones((2, 20011), dtype=np.float32)), 40)  # boundary bucket overflow: radix fallback
_lib.config_set("large_fast", 0)
osmx.softmax_topk(x, 100)  # large k: radix + CUB path
_lib.config_set("large_fast", 1)
big1 = rng.standard_normal((1, 300003)).astype(np.float32)
x1 = dev(big1)[:, 1:]  # misaligned one row
osmx.softmax_topk(x1, 5)  # one row: TMA ring over dynamic chunks + last-CTA merge
osmx.topk(x1, 9)
for cfg in (0, 2):
    _lib.config_set("tma_cfg", cfg)
    osmx.softmax_topk(x1, 5)
_lib.config_set("tma_cfg", -1)
_lib.config_set("split_cta", 2)
osmx.softmax_topk(x1, 5)  # static TMA-ring pieces + combine launch
_lib.config_set("split_cta", 0)
osmx.softmax_topk(x1, 5)  # warp-piece split + combine
osmx.topk(x1, 9)
_lib.config_set("split_cta", -1)
for V in (5623, 7500, 10000):  # staged layouts (2-warp groups up to 8K, <= 4 slots above)
    xs = dev(rng.standard_normal((300, V)).astype(np.float32))
    for alg in ("naive", "safe", "online"):
        osmx.softmax(xs, alg=alg)
torch.cuda.synchronize()
print("sanitize run ok")
