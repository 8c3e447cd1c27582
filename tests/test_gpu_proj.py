"""The projection layer fused with the online softmax + top-K
(osmx_proj_softmax_topk, tcgen05 tensor cores): against the same selection
run on fp32 logits computed by cuBLAS (torch.mm, bf16 in, fp32 out) --
the oracle's online_softmax_topk (the reference algorithm) on those logits.
The two GEMMs round their fp32 accumulation differently, so indices may
differ only where the reference logits tie within 1e-5 relative (counted)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bn", [0, 128, 224, 256])
@pytest.mark.parametrize("rows,D,V,k", [(128, 64, 256, 5), (200, 256, 3000, 5), (129, 520, 4097, 8),
                                        (512, 1024, 32768, 5), (64, 4096, 20000, 32), (300, 128, 700, 1),
                                        (1000, 512, 70000, 5)])
def test_proj_topk_vs_reference_on_fp32_logits(cuda, oracle_mod, rows, D, V, k, bn):
    import torch

    from paper_1805_02867_b200 import _lib, osmx

    _lib.config_set("proj_bn", bn)

    g = torch.Generator(device="cuda")
    g.manual_seed(rows * 7 + V)
    h = (torch.randn((rows, D), device="cuda", generator=g) / D ** 0.25).to(torch.bfloat16)
    w = (torch.randn((V, D), device="cuda", generator=g) / D ** 0.25).to(torch.bfloat16)
    try:
        vals, idx = osmx.proj_softmax_topk(h, w, k)
    finally:
        _lib.config_set("proj_bn", 0)
    z = torch.mm(h, w.t(), out_dtype=torch.float32)
    zc = z.cpu().numpy()
    rv, rz, st = oracle_mod.batch("online_softmax_topk", zc, k=k)
    assert (st == 0).all()
    gi, gv = idx.cpu().numpy(), vals.cpu().numpy()
    diff = 0
    for r in range(rows):
        if not np.array_equal(gi[r], rz[r]):
            a, b = np.sort(zc[r, gi[r]]), np.sort(zc[r, rz[r]])
            assert np.allclose(a, b, rtol=1e-5, atol=1e-6), (r, gi[r], rz[r])
            diff += 1
    assert diff <= max(1, rows // 100)
    rel = np.abs(gv.astype(np.float64) - rv) / rv
    assert rel.max() <= 2e-4, rel.max()  # logits differ by fp32 accumulation order (~1e-6 abs)
    print(f"rows {rows} D {D} V {V} k {k}: index rows differing by logit ties: {diff}, max rel {rel.max():.2e}")


def test_proj_nan_logit_block_flagged(cuda):
    """A whole 32-column chunk of NaN logits (NaN rows of W) must still poison
    the row normalizer: every row is reported non-finite, like the reference
    on those fp32 logits."""
    import torch

    from paper_1805_02867_b200 import osmx

    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    h = torch.randn((130, 256), device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn((1000, 256), device="cuda", generator=g).to(torch.bfloat16)
    w[64:128] = float("nan")
    with pytest.raises(osmx.NonFiniteError) as e:
        osmx.proj_softmax_topk(h, w, 5)
    assert e.value.row == 0
