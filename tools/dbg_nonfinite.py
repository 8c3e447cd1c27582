"""Print every (shape, bad, V, alg) whose non-finite row is not flagged."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1805_02867_b200 import _lib, osmx

_lib.load()
rng = np.random.default_rng(5)
for shape in (0, 1, 2, 3, 4):
    _lib.config_set("shape", shape)
    _lib.config_set("split_chunk", 2048 if shape == 3 else 0)
    for bad in (np.nan, np.inf, -np.inf):
        for V in (7, 3000, 40000):
            if shape in (1, 4) and V > 16384:
                continue
            x = rng.standard_normal((6, V)).astype(np.float32)
            x[4, V // 2] = bad
            x[5, 0] = bad
            for alg in ("naive", "safe", "online"):
                try:
                    osmx.softmax(torch.from_numpy(x).cuda(), alg=alg)
                    print("NOT FLAGGED", shape, bad, V, alg)
                except osmx.NonFiniteError as e:
                    if e.row != 4:
                        print("WRONG ROW", shape, bad, V, alg, e.row)
print("done")
