"""Regression: the staged softmax ring must not hang or fault under many
back-to-back graph-replayed launches.  With one spare ring slot and >= 4
consumer groups -- (D, NG) = (5, 4) ... (8, 7), the former defaults for
6500 < V <= 8192 -- about one launch in 10^3-10^4 hung or faulted on B200
(tools/runs/r2_aq.sh, r2_ar.sh); those layouts are no longer chosen
(csrc/softmax_staged.cuh run_staged_cfg).  Each case replays 2000 launches
in a subprocess under a timeout, so a regression fails instead of hanging
the suite, and checks the result against torch."""
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
    B, V = 4000, {V}
    for key, val in {knobs!r}:
        _lib.config_set(key, val)
    x = torch.randn(2, B, V, device="cuda")
    y = torch.empty_like(x)
    alg = getattr(_lib, {alg!r})
    nb = lib.osmx_workspace_bytes(alg, B, V, 0)
    ws = torch.zeros(max(nb, 256), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for j in range(40):
            st = lib.osmx_softmax(alg, x[j % 2].data_ptr(), V, y[j % 2].data_ptr(), V, B, V, ws.data_ptr(),
                                  ws.numel(), s.cuda_stream)
            assert st == 0
    for _ in range(50):
        g.replay()
    torch.cuda.synchronize()
    ref = torch.softmax(x[1].double(), dim=1)
    err = float(((y[1].double() - ref).abs() / ref).max())
    assert err < 1e-5, err
    print("ok")
""")


@pytest.mark.parametrize("V,knobs,alg", [
    (7000, [], "ONLINE_SOFTMAX"),
    (7500, [], "ONLINE_SOFTMAX"),
    (8000, [], "ONLINE_SOFTMAX"),
    (7500, [], "SAFE_SOFTMAX"),
    (10000, [("staged_ng", 4)], "ONLINE_SOFTMAX"),
    (7500, [("staged_kb", 120)], "ONLINE_SOFTMAX"),
])
def test_staged_ring_many_graph_launches(cuda, V, knobs, alg):
    code = SCRIPT.format(root=str(ROOT), V=V, knobs=knobs, alg=alg)
    try:
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=180)
    except subprocess.TimeoutExpired:
        pytest.fail(f"staged softmax hung under graph replay (V={V}, {knobs})")
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
