"""configs[4] timeline of the one-row dynamic-chunk top-K (split_cta=4):
per-CTA %globaltimer stamps from the OSMX_TIMELINE diagnostic build
(make timeline -> build/tl/libosmx_b200.so).  Prints, per layout, the span
from the first CTA start to the combine end, the spread of CTA starts and
streaming ends, chunks per CTA, and the ticket -> combine time.

    OSMX_LIB_DIAG=build/tl/libosmx_b200.so python tools/c5_timeline.py
"""
import ctypes as C
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ.setdefault("OSMX_LIB_DIAG", str(Path(__file__).resolve().parents[1] / "build/tl/libosmx_b200.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1805_02867_b200 import _lib  # noqa: E402

lib = _lib.load()
lib.osmx_diag_timeline.restype = C.c_int
lib.osmx_diag_timeline.argtypes = [C.c_void_p, C.c_int]
lib.osmx_diag_timeline_clear.restype = C.c_int
lib.osmx_diag_timeline2.restype = C.c_int
lib.osmx_diag_timeline2.argtypes = [C.c_void_p]
V, k = 1 << 26, 5
xs = [torch.randn(V, device="cuda") for _ in range(2)]
vals = torch.empty(k, device="cuda")
idx = torch.empty(k, dtype=torch.int64, device="cuda")
nb = lib.osmx_workspace_bytes(_lib.ONLINE_SOFTMAX_FUSED_TOPK, 1, V, k)
ws = torch.zeros(nb, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
buf = np.zeros(1024 * 5, dtype=np.uint64)
for cfg in (0, 1, 2):
    _lib.config_set("split_cta", 4)
    _lib.config_set("tma_cfg", cfg)
    spans = []
    for rep in range(12):
        lib.osmx_diag_timeline_clear()  # no stale stamps (a layout with fewer CTAs)
        lib.osmx_softmax_topk(_lib.ONLINE_SOFTMAX_FUSED_TOPK, xs[rep % 2].data_ptr(), V, 1, V, k, vals.data_ptr(),
                              idx.data_ptr(), ws.data_ptr(), ws.numel(), st)
        torch.cuda.synchronize()
        buf[:] = 0
        lib.osmx_diag_timeline(buf.ctypes.data, buf.size)
        t = buf.reshape(1024, 5).astype(np.int64)
        n = int((t[:, 0] > 0).sum())
        t = t[:n]
        t0 = t[:, 0].min()
        last = int(np.argmax(t[:, 2]))
        b2 = np.zeros(16, dtype=np.uint64)
        lib.osmx_diag_timeline2(b2.ctypes.data)
        stamps = [(int(v) - int(t0)) / 1e3 if v else None for v in b2[:11]]
        spans.append(((t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, (t[last, 3] - t0) / 1e3,
                      t[:, 4]))
    s0, s1, s2, s3, ch = spans[-1]
    tot = np.array([sp[3] for sp in spans[2:]])
    print(f"tma_cfg={cfg} CTAs={len(s0)}: span(first start -> combine end) median {np.median(tot):.2f} us "
          f"[{tot.min():.2f}, {tot.max():.2f}]")
    print(f"   starts   min/med/max {s0.min():.2f} {np.median(s0):.2f} {s0.max():.2f} us")
    print(f"   stream end min/med/max {s1.min():.2f} {np.median(s1):.2f} {s1.max():.2f} us")
    print(f"   ticket   min/med/max {s2.min():.2f} {np.median(s2):.2f} {s2.max():.2f} us; combine end {s3:.2f} us")
    print("   last CTA: fence in/out", stamps[5], stamps[6], "| loads done", stamps[0], "md/min reduced", stamps[1],
          "warp merge", stamps[2], "sync", stamps[3], "w0 reduced", stamps[7],
          "lists", stamps[8], "final", stamps[4])
    print(f"   chunks/CTA min/med/max {ch.min()} {int(np.median(ch))} {ch.max()}")
