"""configs[4] single row V = 2^26: fused top-5 / online softmax time per knob
setting.  Each argument is one setting, "key=value[,key=value...]"; knobs are
restored to their previous values afterwards."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from bench import measured_peaks, run_c5
from paper_1805_02867_b200 import _lib

lib = _lib.load()
dev = torch.device("cuda", 0)
l2 = torch.cuda.get_device_properties(dev).L2_cache_size
peak = measured_peaks()["hbm_gbs"]
for spec in sys.argv[1:] or ["split_chunk=0"]:
    kvs = [(kv.split("=")[0], int(kv.split("=")[1])) for kv in spec.split(",") if kv]
    old = [(k, _lib.config_get(k)) for k, _ in kvs]
    for k, v in kvs:
        _lib.config_set(k, v)
    r = run_c5(lib, _lib, dev, 15, peak, l2)
    print(spec, json.dumps({k: {kk: r[k][kk] for kk in ("ms", "GBps", "frac")} for k in ("online_fused", "online")}),
          flush=True)
    for k, v in old:
        _lib.config_set(k, v)
