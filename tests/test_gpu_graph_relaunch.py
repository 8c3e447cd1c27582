"""Regression: the staged softmax replayed from CUDA graphs after another
ring layout of the same kernel instantiation ran in the same process.  A
C = 1 launch that carried a (1,1,1) cluster attribute hung in exactly this
sequence (default ring, then staged_kb=120, 4000 x 7500, graph replay;
tools/runs/r2_ah.sh); C = 1 launches now carry no cluster attribute.  Run in
a subprocess under a timeout so a regression fails instead of hanging."""
from __future__ import annotations

import subprocess
import sys
import textwrap
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = textwrap.dedent("""
    import sys
    sys.path.insert(0, {root!r})
    import torch
    from paper_1805_02867_b200 import _lib
    lib = _lib.load()
    B, V = 4000, 7500
    x = torch.randn(2, B, V, device="cuda")
    y = torch.empty_like(x)
    for kb in (0, 120, 0, 160, 120):
        _lib.config_set("staged_kb", kb)
        nb = lib.osmx_workspace_bytes(_lib.ONLINE_SOFTMAX, B, V, 0)
        ws = torch.zeros(max(nb, 256), dtype=torch.uint8, device="cuda")
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for j in range(6):
                st = lib.osmx_softmax(_lib.ONLINE_SOFTMAX, x[j % 2].data_ptr(), V, y[j % 2].data_ptr(), V, B, V,
                                      ws.data_ptr(), ws.numel(), s.cuda_stream)
                assert st == 0
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        ref = torch.softmax(x[1].double(), dim=1)
        assert float(((y[1].double() - ref).abs() / ref).max()) < 1e-5, kb
    _lib.config_set("staged_kb", 0)
    print("ok")
""")


def test_staged_layouts_in_graphs_do_not_hang(cuda):
    code = SCRIPT.format(root=str(ROOT))
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    except subprocess.TimeoutExpired:
        pytest.fail("staged softmax graph replay hung (> 120 s)")
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
