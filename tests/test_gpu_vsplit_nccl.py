"""The NCCL V-split of one huge row through the C-ABI (osmx_vsplit_*):
slice record -> ncclAllGather -> rank-order merge, on the caller's stream.

The box has one GPU, so the communicator has one rank (NCCL refuses two
ranks on one device); the multi-rank merge order is the same code path as
osmx_records_combine over n records, covered by test_gpu_fullsize (8 slices
of the 2^26 row) and, for the gather itself, by the gloo tests in
test_dist.py.  Here: the C-ABI call, its parity with the single-GPU path and
the oracle, the empty slice, non-finite input and CUDA-graph capture."""
from __future__ import annotations

import numpy as np
import pytest

from tests._util import max_rel

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def comm():
    from paper_1805_02867_b200 import osmx

    if not osmx.nccl_available():
        pytest.skip("libnccl.so.2 not loadable")
    c = osmx.NcclComm(1, 0, osmx.NcclComm.unique_id())
    yield c
    c.close()


@pytest.mark.parametrize("V,k", [(1, 1), (37, 5), (70001, 5), (1 << 20, 8), (3 << 20, 32)])
def test_vsplit_topk_matches_oracle(cuda, oracle_mod, comm, V, k):
    import torch

    from paper_1805_02867_b200 import osmx

    if k > V:
        pytest.skip("k > V")
    rng = np.random.default_rng(V + k)
    x = rng.standard_normal(V).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    vals, idx = osmx.vsplit_softmax_topk_nccl(xd, 0, k, comm)
    rv, rz, st = oracle_mod.batch("online_softmax_topk", x[None], k=k)
    assert (st == 0).all()
    assert np.array_equal(idx.cpu().numpy(), rz[0])
    assert max_rel(vals.cpu().numpy()[None], rv) <= TOL
    # the single-GPU path gives the same answer
    sv, si = osmx.softmax_topk(xd[None], k)
    assert torch.equal(si[0], idx)


def test_vsplit_col0_and_softmax(cuda, oracle_mod, comm):
    """col0 shifts the global indices; the softmax leg scales this slice with
    the merged (M, D)."""
    import torch

    from paper_1805_02867_b200 import osmx

    rng = np.random.default_rng(5)
    x = rng.standard_normal(200003).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    vals, idx = osmx.vsplit_softmax_topk_nccl(xd, 1000, 5, comm)
    _, rz, _ = oracle_mod.batch("online_softmax_topk", x[None], k=5)
    assert np.array_equal(idx.cpu().numpy(), rz[0] + 1000)
    y = osmx.vsplit_softmax_nccl(xd, 0, comm).cpu().numpy()
    ry, _ = oracle_mod.batch("online_softmax", x[None])
    assert max_rel(y[None], ry) <= TOL


def test_vsplit_nonfinite_and_capture(cuda, comm):
    import torch

    from paper_1805_02867_b200 import osmx

    x = torch.randn(1 << 20, device="cuda")
    x[12345] = float("nan")
    with pytest.raises(osmx.NonFiniteError):
        osmx.vsplit_softmax_topk_nccl(x, 0, 5, comm)
    x[12345] = 0.0
    ref_v, ref_i = osmx.vsplit_softmax_topk_nccl(x, 0, 5, comm)
    # record -> all-gather -> combine captured in one CUDA graph
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        osmx.vsplit_softmax_topk_nccl(x, 0, 5, comm, check=False)  # workspace for this stream
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            gv, gi = osmx.vsplit_softmax_topk_nccl(x, 0, 5, comm, check=False)
    g.replay()
    torch.cuda.synchronize()
    # indices exact; values to fp32 rounding -- the one-row split assigns
    # chunks to CTAs dynamically, so d's last bits follow the assignment
    assert torch.equal(gi, ref_i) and torch.allclose(gv, ref_v, rtol=1e-6, atol=0)
