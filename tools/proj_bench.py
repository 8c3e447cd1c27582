"""Fused projection + online softmax top-K vs cuBLAS GEMM (fp32 logits in
HBM) + the fused top-K kernel, LM-head shapes; TFLOP/s vs MEASURED_PEAKS."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1805_02867_b200 import _lib, osmx

dev = torch.device("cuda", 0)
peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()).get("bf16_tflops", 1663.0) \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 1663.0


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


for rows, D, V, k in [(4096, 4096, 32768, 5), (4096, 4096, 131072, 5), (1024, 8192, 131072, 5), (128, 4096, 131072, 5),
                      (32, 4096, 131072, 5), (256, 8192, 131072, 5)]:
    h = (torch.randn((rows, D), device=dev) / D ** 0.25).to(torch.bfloat16)
    w = (torch.randn((V, D), device=dev) / D ** 0.25).to(torch.bfloat16)
    flops = 2.0 * rows * V * D
    tf = {}
    for bn in (128, 256):
        _lib.config_set("proj_bn", bn)
        tf[bn] = timeit(lambda: osmx.proj_softmax_topk(h, w, k, check=False))
    _lib.config_set("proj_bn", 0)
    t_f = timeit(lambda: osmx.proj_softmax_topk(h, w, k, check=False))
    t_g = timeit(lambda: torch.mm(h, w.t(), out_dtype=torch.float32))
    z = torch.mm(h, w.t(), out_dtype=torch.float32)
    t_t = timeit(lambda: osmx.softmax_topk(z, k, check=False))
    r = {"rows": rows, "D": D, "V": V, "k": k, "fused_ms": round(t_f, 4), "fused_TFLOPs": round(flops / t_f / 1e9, 1),
         "fused_frac_bf16_peak": round(flops / t_f / 1e9 / peak, 3), "cublas_gemm_fp32out_ms": round(t_g, 4),
         "cublas_TFLOPs": round(flops / t_g / 1e9, 1), "topk_on_logits_ms": round(t_t, 4),
         "unfused_ms": round(t_g + t_t, 4), "fused_over_unfused": round((t_g + t_t) / t_f, 3),
         "by_bn": {b: round(v, 4) for b, v in tf.items()}}
    print(json.dumps(r), flush=True)
    del h, w, z
    torch.cuda.empty_cache()
