"""Same-box FP4 comparators for the bench line (context only, not parity
oracles): library FP4 GEMMs fed THIS path's operands -- K1's E2M1 codes and swizzled scale
factors are the cuBLAS / CUTLASS block-scaled layout, so every library reads the same bytes --
and the paper authors' own Blackwell kernels (QuTLASS, as installed in vLLM).

  cublaslt_fp4      torch._scaled_mm on float4_e2m1fn_x2 operands (cuBLASLt block-scaled GEMM)
  flashinfer_fp4    flashinfer.mm_fp4 (backend auto)
  vllm_cutlass_nvfp4  vllm _custom_ops.cutlass_scaled_fp4_mm (NVFP4)
  qutlass_mxf4      vllm _custom_ops.matmul_mxf4_bf16_tn (QuTLASS, MXFP4)
  qutlass_quant_mx / qutlass_quant_nv   fusedQuantizeMx / fusedQuantizeNv: QuTLASS's rotate +
                    quantize (the K1 counterpart; NVFP4 with a static global scale)

Each entry: {"us": mean flushed-L2 CUDA-event time, "tflops" (GEMMs) or "gbs" (quantizers)}, or
{"error": "..."} when the library or the shape is unavailable.
"""

from __future__ import annotations

import torch


def _time(fn, flush, n, stream):
    for _ in range(3):
        fn()
    ev = []
    for _ in range(n):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        ev.append((e0, e1))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / n * 1e-3


def run(x, a, w, fmt: str, had: int, flush, n: int = 20) -> dict:
    """x: bf16 activations [M, K]; a: GpuQuantResult of x (K1); w: PackedWeight [N, K]."""
    M, K = x.shape
    N = w.N
    flops = 2.0 * M * N * K
    stream = torch.cuda.current_stream()
    out = {}
    G = 32 if fmt == "mxfp4" else 16
    sf_dtype = getattr(torch, "float8_e8m0fnu", None) if fmt == "mxfp4" else torch.float8_e4m3fn
    a4 = a.codes.view(torch.float4_e2m1fn_x2) if hasattr(torch, "float4_e2m1fn_x2") else None
    b4 = w.codes.view(torch.float4_e2m1fn_x2) if a4 is not None else None
    alpha = (a.tensor_scale_dev * w.tensor_scale_dev).contiguous()
    # the swizzled scale-factor buffers as the 2-D [rows padded to 128, K/G padded to 4] matrices
    # the libraries index (the bytes are already their 128x4 block-scaled layout)
    cols = ((K // G) + 3) // 4 * 4
    sa2 = a.sf.view(-1)[:((M + 127) // 128 * 128) * cols].view((M + 127) // 128 * 128, cols)
    sb2 = w.sf.view(-1)[:((N + 127) // 128 * 128) * cols].view((N + 127) // 128 * 128, cols)

    def gemm_entry(name, fn):
        try:
            fn()
            torch.cuda.synchronize()
            t = _time(fn, flush, n, stream)
            out[name] = {"us": t * 1e6, "tflops": flops / t / 1e12}
        except Exception as e:  # noqa: BLE001 - comparators are optional context
            out[name] = {"error": f"{type(e).__name__}: {str(e)[:600]}"}

    if a4 is not None and sf_dtype is not None:
        sa, sb = sa2.view(sf_dtype), sb2.view(sf_dtype)
        if fmt == "nvfp4":   # alpha applied by _scaled_mm's scale_result is not available: fold later
            gemm_entry("cublaslt_fp4", lambda: torch._scaled_mm(a4, b4.t(), sa.view(-1), sb.view(-1),
                                                                out_dtype=torch.bfloat16))
        else:
            gemm_entry("cublaslt_fp4", lambda: torch._scaled_mm(a4, b4.t(), sa.view(-1), sb.view(-1),
                                                                out_dtype=torch.bfloat16))
            if "error" in out["cublaslt_fp4"]:
                gemm_entry("cublaslt_fp4", lambda: torch._scaled_mm(a4, b4.t(), sa, sb, out_dtype=torch.bfloat16))
    try:
        import flashinfer
        sa8 = sa2.view(torch.float8_e4m3fn if fmt == "nvfp4" else torch.uint8)
        sb8 = sb2.view(torch.float8_e4m3fn if fmt == "nvfp4" else torch.uint8)
        gemm_entry("flashinfer_fp4", lambda: flashinfer.mm_fp4(
            a.codes, w.codes.t(), sa8, sb8.t(), alpha, torch.bfloat16, block_size=G, use_nvfp4=fmt == "nvfp4"))
    except Exception as e:  # noqa: BLE001
        out["flashinfer_fp4"] = {"error": f"{type(e).__name__}: {str(e)[:160]}"}
    try:
        import vllm._custom_ops as ops
        if fmt == "nvfp4":
            gemm_entry("vllm_cutlass_nvfp4", lambda: ops.cutlass_scaled_fp4_mm(
                a.codes, w.codes, sa2.view(torch.float8_e4m3fn), sb2.view(torch.float8_e4m3fn), alpha,
                torch.bfloat16))
        else:
            gemm_entry("qutlass_mxf4", lambda: ops.matmul_mxf4_bf16_tn(
                a.codes, w.codes, a.sf.view(torch.float8_e8m0fnu), w.sf.view(torch.float8_e8m0fnu), alpha))
        # QuTLASS rotate + quantize (K1 counterpart): H_k as a dense [k, k] bf16 matrix
        from paper_2509_23202_b200.gptq import _sylvester_unit
        H = _sylvester_unit(had, x.device).to(torch.bfloat16)
        qbytes = M * K * (2 + 0.5 + 1.0 / G)
        try:
            if fmt == "mxfp4":
                fn = lambda: ops.fusedQuantizeMx(x, H, method="abs_max")
            else:
                gs = torch.ones(1, dtype=torch.float32, device=x.device)
                fn = lambda: ops.fusedQuantizeNv(x, H, gs)
            fn()
            torch.cuda.synchronize()
            t = _time(fn, flush, n, stream)
            out["qutlass_quant_" + fmt[:2]] = {"us": t * 1e6, "gbs": qbytes / t / 1e9}
        except Exception as e:  # noqa: BLE001
            out["qutlass_quant_" + fmt[:2]] = {"error": f"{type(e).__name__}: {str(e)[:160]}"}
    except Exception as e:  # noqa: BLE001
        out["vllm"] = {"error": f"{type(e).__name__}: {str(e)[:160]}"}
    return out


if __name__ == "__main__":
    import json
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import paper_2509_23202_b200 as P
    from paper_2509_23202_b200.quantize import act_quant_into, alloc_result
    flush_w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for cfg in sys.argv[1:] or ["c1", "c2-up-nv"]:
        name, M, K, N, fmt, had = bench.CONFIGS[cfg]
        spec = P.FormatSpec.mxfp4() if fmt == "mxfp4" else P.FormatSpec.nvfp4()
        x = torch.randn(M, K, device="cuda").bfloat16()
        w = P.quantize_weight((torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16(), spec,
                              P.TransformSpec.hadamard(had))
        a = alloc_result(M, K, w.fmt, had, "cuda")
        act_quant_into(x, w.fmt, had, a.codes, a.sf, a.tensor_scale_dev, a.scratch)
        res = run(x, a, w, fmt, had, flush_w.zero_)
        y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        ours = _time(lambda: P.gemm(a, w, y), flush_w.zero_, 20, torch.cuda.current_stream())
        res["ours_k2"] = {"us": ours * 1e6, "tflops": 2.0 * M * N * K / ours / 1e12}
        print(cfg, json.dumps(res))
