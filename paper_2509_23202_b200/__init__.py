"""B200-native MR-GPTQ FP4 quantized-linear path (drop-in for microfp's hot path).

Mirrors the reference package's names (/root/reference/pkg/src/microfp/__init__.py:9-61)
for everything on the path ``Q(X H_k) Q(W H_k)^T``:

    quantize_rtn / quantize          K1: fused Hadamard + FP4 quantization (CUDA)
    quantize(policy=MSE)             offline MSE scale search on the GPU (weights)
    FormatSpec, ScaleFormat, ...     format descriptors (same fields as the reference)
    MfpTensor, pack_tensor, ...      host container (interchange with the reference)
    prepare_weight, quantize_weight  K3: weight prep into the tensor-core layout
    quantized_linear                 K1 + K2 (tcgen05 block-scaled FP4 GEMM)
    quantized_linear_host            the same on host buffers, H2D / compute / D2H pipelined
    quantized_linear_requant         K2 + the next layer's MXFP4 act-quant fused in its epilogue
    GraphedLinear                    a fixed-shape quantized_linear captured into a CUDA graph
    gptq.gptq_quantize / mr_gptq     GPU GPTQ / MR-GPTQ solver (offline weights)
    quantized_linear_sharded         N-sharded linear + NCCL all-gather

All compute runs in libmrfp4.so (sm_100a); there is no CPU fallback.
"""

from .errors import DataError, NumericalError
from .fileio import parse_quant, quant_bytes, read_quant, write_quant
from .formats import (FMT_MXFP4, FMT_NVFP4, FormatSpec, MfpTensor, ScaleFormat, ScaleKind, ScaleMode, ScalePolicy,
                      pack_tensor, unpack_tensor)
from .linear import (GraphedLinear, PackedWeight, gemm, prepare_weight, quantize_weight, quantized_linear, quantized_linear_host,
                     quantized_linear_requant)
from .quantize import GpuQuantResult, mse_optimize_scales, quantize, quantize_rtn
from .transforms import TransformKind, TransformSpec

__version__ = "0.1.0"

__all__ = [
    "DataError", "NumericalError", "FormatSpec", "ScaleFormat", "ScaleKind", "ScaleMode", "ScalePolicy", "MfpTensor",
    "mse_optimize_scales",
    "TransformKind", "TransformSpec", "pack_tensor", "unpack_tensor", "quantize_rtn", "quantize",
    "GpuQuantResult", "PackedWeight", "prepare_weight", "quantize_weight", "quantized_linear", "quantized_linear_host", "quantized_linear_requant", "GraphedLinear", "gemm",
    "quantized_linear_sharded", "read_quant", "write_quant", "parse_quant", "quant_bytes",
    "FMT_MXFP4", "FMT_NVFP4",
]


from . import gptq  # noqa: E402


def __getattr__(name):
    if name == "quantized_linear_sharded":
        from .sharded import quantized_linear_sharded
        return quantized_linear_sharded
    raise AttributeError(name)
