"""List (shape, phase, pos, value, alg) combinations whose non-finite row is not reported."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_1805_02867_b200 import _lib, osmx

_lib.load()
SH = {"auto": 0, "resident": 1, "stream": 2, "split": 3, "staged": 4, "cluster": 5}
rng = np.random.default_rng(17)
V = 3001
for shape in ("auto", "staged", "cluster"):
    _lib.config_set("shape", SH[shape]); _lib.config_set("cluster_size", 3 if shape == "cluster" else 0)
    for phase in range(4):
        big = rng.standard_normal((3, V + 4)).astype(np.float32)
        for pos in (0, 1, 2, V - 2, V - 1):
            for bad in (np.nan, np.inf, -np.inf):
                b = big.copy(); b[1, phase + pos] = bad
                xt = torch.from_numpy(b).cuda()[:, phase:phase + V]
                for alg in ("safe", "online"):
                    try:
                        osmx.softmax(xt, alg=alg); print("MISS", shape, phase, pos, bad, alg)
                    except osmx.NonFiniteError as e:
                        if e.row != 1: print("ROW", e.row, shape, phase, pos, bad, alg)
